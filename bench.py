#!/usr/bin/env python
"""Benchmark of the hot path: the full (min,+) power-until-periodic run of A(D_n) (default
n = 12, the paper's largest case) and gamma_2(P_n x C_m) read off from it.

One "step" = one whole run of SURVEY.md section 8(a) rows a2-a6 (stage A, A^k = A (x) A^{k-1}
with fused periodicity statistics until A^{mu+lambda} = b (x) A^mu, read gamma_2) on a device-
resident A.  The metric is BASELINE.json's: (min,+) Gop/s and seconds to gamma_2.  One op =
one add + one min on one 16-bit lane; `value` counts the method's own work, nnz(A) x (columns
computed) per product -- every finite A_il against every computed column (the +inf terms a dense
loop would also visit are reported separately as `dense_equivalent_gops`).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--n 12] [--impl reference]

With --gpus N > 1 and no torchrun environment the script relaunches itself under
torch.distributed.run with N ranks (one per GPU, NCCL all-reduce of the per-power statistics
over NVLink); under torchrun it uses WORLD_SIZE.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
DPX_STEPS_PER_CLK_PER_SM = 128  # 64 VIADDMNMX.U16x2 lanes / clk / SM x 2 steps
KERNEL_NAMES = {"dense": "k_minplus (dense tiles, VIADDMNMX.U16x2)",
                "tiles": "k_minplus (block-sparse tiles, VIADDMNMX.U16x2)",
                "spmm": "k_spmm (grouped SpMM, VIADDMNMX.U16x2)",
                "small": "k_small_run (the whole run in one thread-block-cluster launch, VIADDMNMX.U16x2)"}
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "ncu_traffic.json")
FOLD_NAME = "k_fold (row-inclusion fold, one launch per DAG level)"


def traffic_bytes(kernel: str, n: int, world: int, sym: bool = False, reuse: bool = False):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel, from the
    committed ncu --set full capture of the same configuration (profiles/ncu_traffic.json)."""
    try:
        table = json.load(open(TRAFFIC_PATH))
    except (OSError, ValueError):
        return None
    rec = table.get(f"{kernel.split()[0]}:{kernel.split('(')[1].split(',')[0]}:n{n}:g{world}" + (":sym" if sym else "")
                    + (":reuse" if reuse else ""))
    return rec["bytes_per_launch"] if rec else None


def hbm_peak() -> float:
    """Measured HBM copy bandwidth (MEASURED_PEAKS.json, driver-written), else the profiling
    guide's B200 figure."""
    try:
        return float(json.load(open(PEAKS_PATH))["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return 6450.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--n", type=int, default=12, help="path order (12 = the paper's largest case)")
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    ap.add_argument("--kernel", default="auto", choices=["auto", "dense", "tiles", "spmm"],
                    help="product kernel (all exact): dense tiles, block-sparse tiles, grouped SpMM")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU time of the oracle sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--spmm-width", type=int, default=0,
                    help="SpMM CTA width override (mp_set_spmm_width; 0 = automatic)")
    ap.add_argument("--no-row-reuse", action="store_true",
                    help="do not use the row-inclusion reuse of A(D_n) (the SpMM over every finite entry)")
    ap.add_argument("--no-symmetry", action="store_true",
                    help="do not pass the word-reversal symmetry of A(D_n) (compute every column)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks
class NvmlClockSampler:
    """SM clock and clock-event reasons read through NVML every 5 ms in a thread during the
    timed region (enough samples even for the millisecond-long small-n runs); falls back to
    the nvidia-smi sampler below if NVML is unavailable."""
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, cuda_index: int):
        import pynvml
        self.nv = pynvml
        pynvml.nvmlInit()
        import torch
        p = torch.cuda.get_device_properties(cuda_index)
        bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        self.smax = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        self.sm, self.reasons, self.run = [], set(), False

    def _loop(self):
        nv = self.nv
        while self.run:
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h) \
                    if hasattr(nv, "nvmlDeviceGetCurrentClocksEventReasons") \
                    else nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001 - a failed sample is skipped, not fatal
                pass
            time.sleep(0.005)

    def start(self):
        self.run = True
        self.thread = threading.Thread(target=self._loop, daemon=True)
        self.thread.start()

    def stop(self) -> dict:
        self.run = False
        self.thread.join(timeout=2)
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.smax,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml, 5 ms"}


def make_clock_sampler(cuda_index: int):
    try:
        return NvmlClockSampler(cuda_index)
    except Exception:  # noqa: BLE001 - no NVML: nvidia-smi
        return ClockSampler(cuda_index)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 500 ms during the timed region (a
    tighter period measurably slowed the many short synchronisations of the small-n runs)."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "500"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi's NVML start-up contends with the CUDA driver for a few hundred ms:
            # let it reach its sampling loop before the timed region starts
            t0 = time.time()
            while len(self.lines) < 2 and time.time() - t0 < 5.0:
                time.sleep(0.05)
            self.lines.clear()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------- cpu oracle
def oracle_sample(n: int, target_s: float, A=None) -> dict:
    """The oracle as it stands (oracle_minplus_ikj: the skip-inf triple loop, OpenMP over rows)
    on a bounded sample of the workload: rows 0..R-1 of one product A (x) X of A(D_n), with
    A(D_n) built by the ORACLE (oracle.transition_matrix) -- the product library is never
    loaded on this path.  The loop visits exactly the finite A_il of those rows against every
    column, so the sample's useful steps are nnz(A[:R]) * N (the unit of `value`) and its
    dense-equivalent steps R * N * N.  The cost of the inner loop does not depend on the dense
    right operand's values, so A itself stands in for A^{k-1}."""
    import numpy as np
    import oracle
    if A is None:
        A = oracle.transition_matrix(n)
    N = A.shape[0]
    nnz_row = np.count_nonzero(A != oracle.INF, axis=1)
    R = max(1, min(N, 64))
    t = time.perf_counter()
    oracle.minplus(np.ascontiguousarray(A[:R]), A)
    dt = time.perf_counter() - t
    R2 = int(min(N, max(R, R * target_s / max(dt, 1e-3))))
    t = time.perf_counter()
    oracle.minplus(np.ascontiguousarray(A[:R2]), A)
    dt = time.perf_counter() - t
    useful = float(nnz_row[:R2].sum()) * N
    return {"value": useful / dt / 1e9, "unit": "Gop/s", "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"rows 0..{R2 - 1} of one product A(D_{n}) (x) X, N={N}, A built by oracle.transition_matrix, "
                      f"skip-inf triple loop (oracle_minplus_ikj), {dt:.1f} s; useful steps nnz(A[:{R2}])*N = "
                      f"{useful:.3e}",
            "dense_equivalent_gops": R2 * N * N / dt / 1e9, "seconds": dt, "A": A}


ORACLE_RUNS_PATH = os.path.join(ROOT, "profiles", "r2", "oracle_runs.json")


def oracle_full_runs():
    """Whole oracle runs to gamma_2 (committed measurements, bench_tools/oracle_runs.py and the
    golden-record generator), for context next to the bounded sample."""
    try:
        return json.load(open(ORACLE_RUNS_PATH))
    except (OSError, ValueError):
        return None


def small_l2(N: int) -> bool:
    """True if one power (2*N^2 bytes) is smaller than twice the 126 MB L2."""
    return 2 * N * N < 2 * 126 * 2**20


def workload_config(n: int, N: int, world: int) -> dict:
    """The config keys both arms report for the same workload."""
    return {"workload": f"P_{n} x C_m: power-until-periodic run of A(D_{n}), N={N}, gamma_2 read-off",
            "n": n, "N": N, "parallelism": f"column shards x{world}" if world > 1 else "single GPU",
            "l2": ("L2 flushed between steps (512 MB write, untimed): each power 2*N^2 = %.3f GB fits in the "
                   "126 MB L2" if small_l2(N) else "inputs larger than L2 (each power 2*N^2 = %.2f GB > 126 MB)")
                  % (2 * N * N / 1e9),
            "ops": "useful: nnz(A) x computed columns per product (one op = add+min on one u16 lane)"}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    """The reference arm of this tier: the CPU oracle (no reference package exists), timed as it
    stands on the host cores; rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    A = oracle.transition_matrix(args.n)
    N = A.shape[0]
    steps = []
    base = None
    per_step = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    for i in range(args.warmup + args.steps):
        b = oracle_sample(args.n, per_step, A)
        if i >= args.warmup:
            steps.append(b)
        base = b
    val = statistics.median(s["value"] for s in steps)
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "Gop/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": statistics.median(s["seconds"] for s in steps) * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u16",
            "data": "synthetic: deterministic transfer matrix A(D_n) (oracle.transition_matrix)",
            "config": dict(workload_config(args.n, N, 1), kernel="oracle (CPU, bounded sample)"),
            "cpu_baseline": {"value": val, "unit": "Gop/s", "cores": base["cores"], "kind": "oracle",
                             "sample": base["sample"], "cpu": cpu_model()},
            "dense_equivalent_gops": statistics.median(s["dense_equivalent_gops"] for s in steps),
            "oracle_full_runs": oracle_full_runs(),
            "e2e": {"value": val, "unit": "Gop/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------- mine
def run_mine(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2409_17688_b200 as mp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        mp.dist_set_torch()
    mp.set_options(args.kernel)
    # A(D_n) is invariant under reversing every word (the path's reflection): the library
    # then computes only the columns g <= sigma(g) and verifies the hint on the device
    mp.set_symmetry(None if args.no_symmetry else mp.word_reversal(args.n))
    # A is A(D_n): the library verifies that on the device and then uses the row-inclusion
    # reuse; --no-row-reuse times the plain grouped SpMM instead
    mp.set_transfer_hint(args.n)
    mp.set_row_reuse(not args.no_row_reuse)
    mp.set_spmm_width(args.spmm_width)
    stream = torch.cuda.current_stream()
    mp.set_stream(stream)

    A = mp.build_transition_matrix(args.n)
    N = A.shape[0]
    nnz = int(np.count_nonzero(A != mp.MP_INF))
    # resident input for the device-timed value; rows padded to 64 columns (128-byte aligned
    # rows: the library's vectorised range / transfer-hint check reads them 16 bytes per lane)
    ldA = -(-N // 64) * 64
    dA = torch.full((N, ldA), -1, dtype=torch.int16, device="cuda")[:, :N]
    dA.copy_(torch.from_numpy(A.view(np.int16)))

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    for _ in range(args.warmup):
        res = mp.minplus_power_until_periodic_device(dA)
    torch.cuda.synchronize()

    clocks = make_clock_sampler(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    launches0 = mp.kernel_launches()
    prod_ms, prod_launches, dense, issued, spmm_ms = 0.0, 0, 0.0, 0.0, 0.0
    stats_ms, total_lib_ms, setup_ms = 0.0, 0.0, 0.0
    # Small powers fit in the 126 MB L2: flush it between steps (a 512 MB write, excluded from
    # the timing by per-step events); large powers exceed it anyway.
    flush = torch.empty(512 * 2**20 // 4, dtype=torch.int32, device="cuda") if small_l2(N) else None
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for s_i in range(args.steps):
        if flush is not None:
            flush.fill_(s_i)
        ev[s_i][0].record(stream)
        res = mp.minplus_power_until_periodic_device(dA)
        ev[s_i][1].record(stream)
        p = mp.last_profile()
        prod_ms += p["product_ms"]
        spmm_ms += p["spmm_ms"]
        prod_launches += p["product_launches"]
        kernel_used = p["kernel"]
        spmm_cols = p["spmm_cols"]
        local_cols, ld = p["local_cols"], p["ld"]
        row_levels, row_parents = p["row_levels"], p["row_parents"]
        fold_bytes = p["fold_bytes"]
        dense += p["dense_steps"]
        issued += p["issued_steps"]
        setup_ms = p["setup_ms"]
        stats_ms += p["stats_ms"]
        total_lib_ms += p["total_ms"]
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    launches = mp.kernel_launches() - launches0
    ms = sum(a.elapsed_time(b) for a, b in ev)

    # e2e: the public host-buffer entry point, A copied from pinned host memory every step
    pinned = torch.from_numpy(A.view(np.int16)).pin_memory()
    Ah = pinned.numpy().view(np.uint16)
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else args.steps
    mp.minplus_power_until_periodic(Ah)  # warm-up of the host-buffer path (its staging buffer)
    barrier()
    torch.cuda.synchronize()
    fev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(e2e_steps)]
    h2d = d2h = 0
    for s_i in range(e2e_steps):
        if flush is not None:
            flush.fill_(s_i)
        fev[s_i][0].record(stream)
        r2 = mp.minplus_power_until_periodic(Ah)
        fev[s_i][1].record(stream)
        p = mp.last_profile()
        h2d += p["h2d_bytes"]
        d2h += p["d2h_bytes"]
        e2e_setup_ms = p["setup_ms"]
    torch.cuda.synchronize()
    barrier()
    e2e_ms = sum(a.elapsed_time(b) for a, b in fev)
    assert (r2.mu, r2.lam, r2.offset) == (res.mu, res.lam, res.offset)

    # SURVEY.md section 8(d) "seconds to gamma_2": a cold gamma2_cylinder(n, 1000) call (no
    # cached record, no workspace), wall clock: word masks on the host, A(D_n) built on the
    # device, the whole power run, the read-off
    mp.shutdown()
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g2_1000 = mp.gamma2_cylinder(args.n, 1000)
    torch.cuda.synchronize()
    g2_seconds = time.perf_counter() - t0
    assert g2_1000 == res.gamma2(1000)
    barrier()

    # the method's own work per product on this rank: every finite A_il against every column the
    # rank computes (with the word-reversal symmetry: its shard of the domain g <= sigma g)
    # (powers past the first repeat that a small-N batch computed anyway are not counted)
    useful = float(nnz) * local_cols * (res.k_last - 1) * args.steps
    vals = torch.tensor([ms, e2e_ms, dense, issued, useful, prod_ms, float(prod_launches), float(launches),
                         float(h2d), float(d2h)], dtype=torch.float64, device="cuda")
    if world > 1:
        mx = vals[:2].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = vals[2:5].clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        vals[:2], vals[2:5] = mx, sm
    ms, e2e_ms, dense_all, issued_all, useful_all = [float(v) for v in vals[:5].tolist()]
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    products = res.k_last - 1
    value = useful_all / (ms * 1e-3) / 1e9
    sm_mhz = clk.get("sm_mhz") or 1965.0
    peak = 148 * DPX_STEPS_PER_CLK_PER_SM * sm_mhz * 1e6 / 1e9  # Gstep/s at the observed clock
    avg_launch_ms = prod_ms / max(1, prod_launches)        # one product: SpMM (+ fold passes)
    avg_kernel_ms = spmm_ms / max(1, prod_launches)        # the product kernel alone
    issued_per_launch = issued / max(1, prod_launches)
    useful_per_launch = float(nnz) * local_cols
    # physical roofline: DPX steps the kernel issued per launch / its duration
    achieved = issued_per_launch / (avg_kernel_ms * 1e-3) / 1e9 if issued_per_launch else None
    # the method's work (every finite A_il x every computed column) / the whole product's time
    useful_rate = useful_per_launch / (avg_launch_ms * 1e-3) / 1e9
    # The roofline of the dominant kernel.  With the row-inclusion reuse k_spmm issues few DPX
    # steps and is bound by HBM: achieved = its ALGORITHMIC bytes per launch (read the X rows
    # once, the sparse form's entries once, write C once: 2 N ld + 32 B x entries) / its
    # duration, against the measured copy bandwidth; traffic = what ncu measured (the X rows
    # staged once per tile that needs them).  Without the reuse it is DPX-issue-bound.
    traffic = traffic_bytes(KERNEL_NAMES[kernel_used], args.n, world, not args.no_symmetry, bool(row_levels))
    alu = {"achieved": achieved, "peak": peak, "unit": "Gstep/s", "frac": (achieved / peak) if achieved else None,
           "issued_steps_per_launch": issued_per_launch or None,
           "work": "issued DPX steps per launch (4-row groups x entries x columns) / CUDA-event duration",
           "peak_source": f"148 SM x 128 steps/clk/SM x {sm_mhz:.0f} MHz observed (DESIGN.md)"}
    common = {"kernel": KERNEL_NAMES[kernel_used], "avg_kernel_ms": avg_kernel_ms, "traffic": traffic,
              "useful_steps_per_product": useful_per_launch, "avg_product_ms": avg_launch_ms,
              "useful_achieved": useful_rate, "useful_frac": useful_rate / peak,
              "useful_note": "nnz(A) x computed columns per product / product time (kernel + fold passes); "
                             "above 1 only when the row-inclusion reuse skips redundant terms",
              "kernel_share_of_step": spmm_ms / max(ms, 1e-9), "product_share_of_step": prod_ms / max(ms, 1e-9)}
    others = []
    if row_levels and kernel_used == "spmm":
        entries = issued_per_launch / (4.0 * ld) if ld else 0.0
        alg_bytes = 2.0 * N * ld * 2 + 32.0 * entries
        hbm = hbm_peak()
        ach = alg_bytes / (avg_kernel_ms * 1e-3) / 1e9
        roofline = dict(common, bound="hbm", achieved=ach, peak=hbm, unit="GB/s", frac=ach / hbm,
                        algorithmic_bytes_per_launch=alg_bytes,
                        bytes_note="read X_{k-1} (N x ld u16) once + write A^k (N x ld) once + the sparse "
                                   "form's 32-byte entries once", peak_source="MEASURED_PEAKS.json hbm_gbs",
                        traffic_GBps=(traffic / (avg_kernel_ms * 1e-3) / 1e9) if traffic else None, alu=alu)
        # The fold passes of the reuse (k_fold, one launch per DAG level) take as long as the SpMM
        # or longer: the roofline object names whichever of the two took more of the step, the
        # other goes to roofline_others.  k_fold's algorithmic bytes per product (summed over its
        # levels' launches): every folded row read and written once, each distinct parent row of
        # a level read once by that level's launch (library-computed from the DAG).
        fold_ms = (prod_ms - spmm_ms) / max(1, prod_launches)  # per product, all its levels
        if fold_bytes and fold_ms > 0:
            fach = fold_bytes / (fold_ms * 1e-3) / 1e9
            ftraffic = traffic_bytes(FOLD_NAME, args.n, world, not args.no_symmetry, True)
            fold = {"kernel": FOLD_NAME, "bound": "hbm", "achieved": fach, "peak": hbm, "unit": "GB/s",
                    "frac": fach / hbm, "traffic": ftraffic, "avg_kernel_ms": fold_ms,
                    "launches_per_product": row_levels - 1, "algorithmic_bytes_per_product": fold_bytes,
                    "bytes_note": "per product over its row_levels - 1 launches: every folded row read + written "
                                  "once, each distinct parent row of a level read once (x ld x 2 B)",
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                    "traffic_GBps": (ftraffic / (fold_ms * 1e-3) / 1e9) if ftraffic else None,
                    "kernel_share_of_step": (prod_ms - spmm_ms) / max(ms, 1e-9)}
            if fold_ms > avg_kernel_ms:
                roofline, others = fold, [roofline]
            else:
                others = [fold]
    else:
        if not achieved:  # the fused small-N run issues no separate product kernel
            alu.update(achieved=useful_rate, frac=useful_rate / peak,
                       work="useful steps per product / the fused run's time per product")
        roofline = dict(common, bound="alu", **{k: v for k, v in alu.items()})
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = oracle_sample(args.n, args.cpu_seconds)
        cpu = {k: v for k, v in cpu.items() if k not in ("seconds", "A")}
        cpu["cpu"] = cpu_model()
        cpu["full_runs"] = oracle_full_runs()
    line = {
        "metric": METRIC, "value": value, "unit": "Gop/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u16",
        "data": "synthetic: deterministic transfer matrix A(D_n) built on the host (no randomness, no datasets)",
        "config": dict(workload_config(args.n, N, world), products_per_step=products, nnz_A=nnz,
                       mu_lambda_b=[res.mu, res.lam, res.offset], gamma2_m1000=res.gamma2(1000),
                       kernel=args.kernel, spmm_cta_cols=spmm_cols or None, cols_rank0=local_cols, ld_rank0=ld,
                       symmetry="none" if args.no_symmetry else "word reversal (columns g <= sigma g computed)",
                       row_reuse=(f"{row_levels} levels, {row_parents} parent links" if row_levels else "off")),
        "seconds_to_gamma2": ms / args.steps / 1e3,
        "dense_equivalent_gops": dense_all / (ms * 1e-3) / 1e9,
        "issued_gops": issued_all / (ms * 1e-3) / 1e9,
        "roofline": roofline,
        "roofline_others": others or None,
        "cpu_baseline": cpu,
        "e2e": {"value": useful_all / args.steps * e2e_steps / (e2e_ms * 1e-3) / 1e9, "unit": "Gop/s",
                "h2d_bytes_per_step": int(h2d / max(1, e2e_steps)), "d2h_bytes_per_step": int(d2h / max(1, e2e_steps)),
                "seconds_to_gamma2": e2e_ms / e2e_steps / 1e3,
                "setup_ms_last_step": e2e_setup_ms},
        "gamma2_cylinder": {"n": args.n, "m": 1000, "gamma2": g2_1000, "seconds_cold_wall": g2_seconds,
                            "note": "words source, word-reversal symmetry, includes allocation"},
        "setup_ms": setup_ms,
        "breakdown_ms_per_step": {"products": prod_ms / args.steps, "product_kernel": spmm_ms / args.steps,
                                  "folds": (prod_ms - spmm_ms) / args.steps, "stats": stats_ms / args.steps,
                                  "setup": setup_ms, "library_total": total_lib_ms / args.steps,
                                  "step": ms / args.steps},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def relaunch_distributed(n_gpus: int) -> int:
    """--gpus N > 1 without a torchrun environment: run this script under torch.distributed.run
    with N ranks on this node (rendezvous on 127.0.0.1) and return its exit code."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n_gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_distributed(args.gpus))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_mine(args)


if __name__ == "__main__":
    main()
