"""Builds libminplus.so variants with -D overrides into bench_tools/variants/<name>.so
(for bench_tools/r2/gpu_ab.sh).  Usage: build_variants.py name=-DA=1,-DB=2 ..."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_17688_b200 import _build  # noqa: E402

out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "variants")
os.makedirs(out, exist_ok=True)
procs = []
for spec in sys.argv[1:]:
    name, defs = spec.split("=", 1)
    cmd = [_build.NVCC, *_build.NVCC_FLAGS, *defs.split(","), "-I" + os.path.join(_build.ROOT, "include"),
           "-o", os.path.join(out, name + ".so"), *_build.sources()]
    procs.append(subprocess.Popen(cmd))
for p in procs:
    assert p.wait() == 0
