"""Reader of tests/golden/oracle_bench_values.txt (written by
tools/make_golden_bench.py from the oracle only)."""
import os

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "oracle_bench_values.txt")


def table():
    d = {}
    with open(PATH) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            name, dtype, n, hx, val = line.split()
            d[name] = {"dtype": dtype, "n": int(n), "hex": hx, "value": float(val)}
    return d


def hex_of(name):
    return table()[name]["hex"]
