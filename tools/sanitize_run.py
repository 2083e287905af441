"""Dev tool: a small run of every kernel path, for compute-sanitizer.

    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_run.py

Covers: split kernel (small n), persistent stream kernel (TMA ring, stash,
batched group levels, last-arriver combine) incl. a ragged tail and the exact
fallback (special values), column kernels (PipeLoader and stream, rows > T with
the column combine), host streaming, complex view, cr top.  Checks bits
against the oracle."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import nrmf_inputs as gen  # noqa: E402
import oracle  # noqa: E402
import paper_2509_06220_b200 as nrmf  # noqa: E402

bad = 0


def check(got, exp, dt, what):
    global bad
    ok = np.asarray(got, dtype=dt).tobytes() == np.asarray(exp, dtype=dt).tobytes()
    bad += not ok
    print(what, "OK" if ok else "MISMATCH", flush=True)


for dt in (np.float64, np.float32):
    for n in (1, 4097, 20 * 4096 + 3, 700 * 4096 + 5):
        x = gen.normal(5, n, dtype=dt)
        check(nrmf.norm(torch.from_numpy(x).cuda()).cpu().numpy(), oracle.nrmf(x), dt, f"norm {dt.__name__} {n}")
    x = gen.normal(6, 700 * 4096, dtype=dt)
    x[12345] = np.inf if dt == np.float64 else np.float32(1e-40)       # exact-path fallback
    check(nrmf.norm(torch.from_numpy(x).cuda()).cpu().numpy(), oracle.nrmf(x), dt, f"norm special {dt.__name__}")
    check(nrmf.norm(torch.from_numpy(x).cuda(), top="cr").cpu().numpy(), oracle.nrmf(x, top="cr"), dt,
          f"norm cr {dt.__name__}")
    for (r, c, ld) in ((4096, 40, 4096), (5000, 9, 5003), (100, 33, 100)):
        A = gen.normal(7, ld * c, dtype=dt)
        At = torch.from_numpy(A).cuda().as_strided((r, c), (1, ld))
        col, fr = nrmf.cols(At)
        ecol, efr = oracle.cols(A, r, c, ld)
        check(col.cpu().numpy(), ecol, dt, f"cols {dt.__name__} {r}x{c} ld {ld}")
        check(fr.cpu().numpy(), efr, dt, f"frob {dt.__name__} {r}x{c} ld {ld}")
    xh = gen.normal(8, 3 * 4096 * 512 + 9, dtype=dt)
    check(nrmf.norm(torch.from_numpy(xh).pin_memory()).numpy(), oracle.nrmf(xh), dt, f"host {dt.__name__}")
print("ALL OK" if bad == 0 else f"{bad} MISMATCHES")
sys.exit(1 if bad else 0)
