"""The C ABI used from plain C (examples/nrmf_example.c: cudaMalloc, nrmf_d on
a user stream, no Python or torch in the process): builds the example with
gcc against include/nrmf.h and libnrmf.so and checks the printed bits against
the oracle."""
import os
import subprocess

import numpy as np
import pytest

import nrmf_inputs as gen
import oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    from paper_2509_06220_b200 import _build
    lib = _build.build()
    out = str(tmp_path_factory.mktemp("cex") / "nrmf_example")
    cuda = "/usr/local/cuda"
    subprocess.check_call(["gcc", "-O2", "-I", os.path.join(ROOT, "include"), "-I", f"{cuda}/include",
                           os.path.join(ROOT, "examples", "nrmf_example.c"), "-o", out,
                           "-L", os.path.dirname(lib), "-l:libnrmf.so", "-L", f"{cuda}/lib64", "-lcudart",
                           f"-Wl,-rpath,{os.path.dirname(lib)}", f"-Wl,-rpath,{cuda}/lib64"])
    return out


@pytest.mark.parametrize("n", [1, 4097, 3 * 4096 * 8 + 11, (1 << 22) + 3])
def test_c_example_matches_oracle(exe, tmp_path, n):
    x = gen.normal(n, n, dtype=np.float64)
    f = tmp_path / "x.f64"
    x.tofile(f)
    r = subprocess.run([exe, str(n), str(f)], capture_output=True, text=True, check=True).stdout
    bits = r.split("bits=")[1].split()[0]
    exp = np.asarray(oracle.nrmf(x), dtype=np.float64).view(np.uint64).item()
    assert int(bits, 16) == exp, r
