"""Dev check: fp64 beyond 2^31 elements (16 GiB, n = 2^31 + 12345): device,
host-streamed and cr-top results against the oracle, relerr vs the exact norm.
(~70 s, most of it the CPU oracle; not part of the test suite.)"""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import nrmf_inputs as gen, oracle
import paper_2509_06220_b200 as nrmf
n = (1 << 31) + 12345
t0 = time.time()
host = torch.empty(n, dtype=torch.float64).pin_memory()
gen.normal(7, n, dtype=np.float64, out=host.numpy())
x = host.to("cuda")
r = nrmf.norm(x).item()
rh = nrmf.norm(host).item()           # host-streamed path
rc = nrmf.norm(x, top="cr").item()
o = oracle.nrmf(host.numpy())
oc = oracle.nrmf(host.numpy(), top="cr")
ex = oracle.exact(host.numpy())
print(dict(n=n, gpu=r.hex(), host=rh.hex(), oracle=float(o).hex(), same=(r == o and rh == o),
           cr_same=(rc == float(oc)), relerr_eps=oracle.relerr(r, ex, np.float64), s=round(time.time() - t0, 1)))
