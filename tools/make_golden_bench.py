#!/usr/bin/env python
"""Write tests/golden/oracle_bench_values.txt: the ORACLE's value (big-endian
hex, as bench.py prints result_hex) of each bench workload, seed 1.  Calls
only oracle/ and the seeded input generators (nrmf_inputs) -- never the CUDA
path -- so bench.py and the GPU tests can check a run of any GPU count
against the same-tree oracle without re-running it (~15 s per 2^30 array)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import nrmf_inputs as gen  # noqa: E402
import oracle  # noqa: E402

WORKLOADS = {
    # name: (generator, n, dtype)
    "c3": (gen.normal, 1 << 30, np.float64),     # C3: DNRMF n=2^30 N(0,1) (bench.py default)
    "c2": (gen.sme, 1 << 30, np.float32),        # SNRMF n=2^30, C2 recipe (bench.py --config c2)
    "c1": (gen.uniform_pm1, 1 << 20, np.float64),  # C1: DNRMF n=2^20 U[-1,1)
}


def main():
    out = os.path.join(ROOT, "tests", "golden", "oracle_bench_values.txt")
    lines = ["# oracle.nrmf (same-tree C oracle, top=v1) of bench.py's workloads, seed 1, offset 0;",
             "# big-endian hex of the IEEE value.  Written by tools/make_golden_bench.py (oracle only)."]
    for name, (g, n, dt) in WORKLOADS.items():
        x = g(1, n, 0, dtype=dt)
        v = np.asarray(oracle.nrmf(x), dtype=dt)
        lines.append(f"{name} {np.dtype(dt).name} {n} {v.tobytes()[::-1].hex()} {float(v)!r}")
        print(lines[-1], flush=True)
        del x
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
