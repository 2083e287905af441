"""Dev tool: run the fast-path checks of a fastcheck .so variant."""
import ctypes
import sys
L = ctypes.CDLL(sys.argv[1])
L.fastcheck.argtypes = [ctypes.c_int, ctypes.c_ulonglong, ctypes.c_ulonglong, ctypes.c_int, ctypes.POINTER(ctypes.c_ulonglong)]
for which, n, mode in [(1, 1 << 28, 0), (1, 1 << 28, 1), (3, int(sys.argv[2]) if len(sys.argv) > 2 else 512, 0)]:
    out = (ctypes.c_ulonglong * 3)()
    rc = L.fastcheck(which, 7, n, mode, out)
    print(which, n, mode, "rc", rc, "checked", out[0], "fast", out[1], "mism", out[2], flush=True)
