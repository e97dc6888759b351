"""Markdown table of bench.py JSON lines (one file per configuration).

    python bench_tools/summarize.py profiles/r1_bench_n*_final.jsonl
"""
import json
import sys


def main(paths):
    print("| n | N | kernel | seconds to gamma_2 | ms / product | issued Gstep/s | roofline frac | "
          "dense-equiv Gop/s | e2e s | setup ms | clocks MHz |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for p in paths:
        lines = [l for l in open(p) if l.startswith("{")]
        if not lines:
            continue
        d = json.loads(lines[-1])
        r, c = d["roofline"], d["config"]
        print(f"| {c['n']} | {c['N']} | {r['kernel'].split('(')[1].split(',')[0]} | {d['seconds_to_gamma2']:.4f} | "
              f"{r['avg_launch_ms']:.3f} | {r['achieved']:.0f} | {r['frac']:.3f} | {d['value']:.0f} | "
              f"{d['e2e']['seconds_to_gamma2']:.4f} | {d.get('setup_ms', 0):.1f} | {d['clocks'].get('sm_mhz')} |")


if __name__ == "__main__":
    main(sys.argv[1:])
