"""Whole oracle runs to gamma_2 on the host cores (SURVEY.md section 8(d) "Timing the oracle
beside it"): Algorithm 2 to the first repeat with the literal triple loop (dense,
n <= DENSE_MAX) and with the skip-inf loop (n <= SKIP_MAX), then gamma_2(P_n x C_1000).

    python bench_tools/oracle_runs.py [out.json] [DENSE_MAX] [SKIP_MAX]

Imports only oracle/ (the CPU checker); writes JSON (default profiles/r2/oracle_runs.json).
The golden-record generator's runs (tests/golden/power_records_n*.json: skip-inf, plus
fingerprints and SHA-256 of every power) are appended as measured on their own host.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402


def cpu_model():
    for line in open("/proc/cpuinfo"):
        if line.startswith("model name"):
            return line.split(":", 1)[1].strip()
    return "unknown"


def run(n, literal):
    A = oracle.transition_matrix(n)
    t0 = time.time()
    P = {1: A}
    k = 1
    while True:  # forward first repeat, every stored power compared (as oracle_power_until_periodic)
        k += 1
        P[k] = oracle.minplus(A, P[k - 1], literal=literal)
        hit = None
        for j in range(k - 1, 0, -1):
            c = oracle.constant_difference(P[k], P[j])
            if c is not None:
                hit = (j, k - j, c)
                break
        if hit:
            break
    mu, lam, b = hit
    diag = [None] + [int(P[i].diagonal().min()) for i in range(1, k + 1)]
    m = 1000
    t = -(-(m - k) // lam)
    g = diag[m - t * lam] + t * b
    return {"n": n, "N": int(A.shape[0]), "loop": "dense ijk (literal)" if literal else "skip-inf ikj",
            "seconds": round(time.time() - t0, 2), "products": k - 1, "mu_lambda_b": [mu, lam, b],
            "gamma2_m1000": g}


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r2", "oracle_runs.json")
    dense_max = int(sys.argv[2]) if len(sys.argv) > 2 else 9
    skip_max = int(sys.argv[3]) if len(sys.argv) > 3 else 10
    res = {"host": cpu_model(), "cores": oracle.num_threads(), "runs": []}
    for n in range(3, skip_max + 1):
        for literal in ([True, False] if n <= dense_max else [False]):
            r = run(n, literal)
            res["runs"].append(r)
            print(json.dumps(r), flush=True)
    gold = []
    for n in (10, 11, 12):
        p = os.path.join(ROOT, "tests", "golden", f"power_records_n{n}.json")
        if os.path.exists(p):
            g = json.load(open(p))
            gold.append({"n": n, "loop": "skip-inf ikj + per-power fingerprint and SHA-256",
                         "seconds": g["seconds"], "threads": g["threads"], "products": g["k_last"] - 1,
                         "host": "the 8-core build container (tests/golden/make_power_records.py)"})
    res["golden_generation"] = gold
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
