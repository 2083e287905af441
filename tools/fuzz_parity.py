"""Dev tool: randomized parity sweep -- N random sizes in [1, 2^24] (log-uniform),
random dtype, distribution, pointer offset (alignment) and top, and (with
--launch) random persistent-grid size, warp-group size and CTA combine step
on/off; GPU vs the oracle bit for bit.  Complements the fixed-size tests."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import nrmf_inputs as gen  # noqa: E402
import oracle  # noqa: E402
import paper_2509_06220_b200 as nrmf  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 300
LAUNCH = "--launch" in sys.argv
SEED = next((int(a.split("=")[1]) for a in sys.argv if a.startswith("--seed=")), 2026)
rng = np.random.default_rng(SEED)
bad = 0
for i in range(N):
    n = int(np.exp(rng.uniform(0, np.log(1 << 24))))
    dt = np.float64 if rng.integers(2) else np.float32
    dist = ["normal", "uniform", "sme", "extreme"][rng.integers(4)]
    if dist == "extreme" and dt != np.float64:
        dist = "sme"
    off = int(rng.integers(0, 4))           # elements of offset: 0 keeps 16-byte alignment only sometimes
    top = "cr" if rng.integers(8) == 0 else "v1"
    seed = int(rng.integers(1, 1 << 30))
    m = n + off
    if dist == "extreme":
        x = gen.extreme(seed, m, ["lit", "fin", "fin2"][seed % 3])
    else:
        x = {"normal": gen.normal, "uniform": gen.uniform_pm1, "sme": gen.sme}[dist](seed, m, dtype=dt)
    xd = torch.from_numpy(x).cuda()[off:]
    grid = g0 = -1
    cta = True
    if LAUNCH:
        grid = int(rng.choice([0, 1, 2, 3, 7, 16, 37, 148, 296]))
        g0 = int(rng.integers(-1, 5))
        cta = bool(rng.integers(4))
        nrmf._debug_set_split_ll(bool(rng.integers(4)))
        nrmf._debug_set_grid(grid)
        nrmf._debug_set_g0(g0)
        nrmf._debug_set_cta_step(cta)
    r = nrmf.norm(xd, top=top).cpu().numpy()
    if LAUNCH:
        nrmf._debug_set_grid(0)
        nrmf._debug_set_g0(-1)
        nrmf._debug_set_cta_step(True)
        nrmf._debug_set_split_ll(True)
    e = oracle.nrmf(x[off:], top=top)
    ok = np.asarray(r, dtype=dt).tobytes() == np.asarray(e, dtype=dt).tobytes()
    if not ok:
        bad += 1
        print("MISMATCH", n, dt.__name__, dist, off, top, seed, grid, g0, cta, flush=True)
print(f"{N} cases, {bad} mismatches")
sys.exit(1 if bad else 0)
