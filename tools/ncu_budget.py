"""Dev tool: per-warp-node instruction budget of the DNRMF/SNRMF kernel from an
ncu --set full capture (source page, SASS), VERDICT r1 item 4.

    python tools/ncu_budget.py report.ncu-rep n_elements [--json out.json --key fp64]

For every SASS instruction ncu reports the warp-level instructions executed
and the stall samples.  They are summed by opcode class over the whole kernel
and divided by the warp-nodes of the call ((n-1)/32: one v1_hypot node per
element bar one, 32 lanes per warp instruction), which gives the executed
instructions per warp-node; the register-file read cycles are estimated per
instruction from its distinct source registers (the bank model of DESIGN.md
§8: cost = max(1, reads of the busier of the two banks)) and summed the same
way."""
import argparse
import collections
import csv
import io
import json
import re
import subprocess


def classify(op):
    o = op.split(".")[0]
    if o in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX"):
        return "fp64"
    if o == "MUFU":
        return "mufu"
    if o in ("FSEL", "SEL"):
        return "select"
    if o in ("FFMA", "FFMA2", "FMUL", "FMUL2", "FADD", "FMNMX", "FSETP"):
        return "fp32"
    if o in ("LDS", "STS", "LDSM"):
        return "smem"
    if o in ("LDG", "STG", "LD", "ST", "ATOM", "ATOMG", "RED", "UBLKCP", "UTMALDG", "SYNCS"):
        return "gmem/async"
    if o in ("BRA", "BSSY", "BSYNC", "EXIT", "CALL", "RET", "WARPSYNC", "BAR", "YIELD", "NOP", "ELECT"):
        return "control"
    return "int/other"


def bank_cycles(text):
    regs = set(re.findall(r"\bR(\d+)\b", text.split(",", 1)[1] if "," in text else ""))
    # a double operand Rk names the pair (Rk, Rk+1)
    op = text.split()[0] if text.split() else ""
    wide = op.startswith(("DFMA", "DMUL", "DADD", "DSETP"))
    even = odd = 0
    for r in regs:
        r = int(r)
        if wide:
            even += 1
            odd += 1
        elif r % 2 == 0:
            even += 1
        else:
            odd += 1
    return max(1, even, odd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("n", type=int)
    ap.add_argument("--json")
    ap.add_argument("--key")
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ci, cs, cst = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    by = collections.Counter()
    stalls = collections.Counter()
    rf = 0.0
    total = 0
    fp64_ops = collections.Counter()
    for r in rows[2:]:
        if len(r) <= ci:
            continue
        try:
            k = int(r[ci])
        except ValueError:
            continue
        text = r[cs].strip()
        op = text.split()[0] if text else "?"
        if op.startswith("@"):
            op = text.split()[1]
            text = " ".join(text.split()[1:])
        c = classify(op)
        by[c] += k
        total += k
        stalls[c] += int(r[cst] or 0)
        rf += k * bank_cycles(text)
        if c == "fp64":
            fp64_ops[op.split(".")[0]] += k
    wn = (a.n - 1) / 32
    print(f"{a.rep}: {total} warp-instructions executed, {wn:.4g} warp-nodes -> {total / wn:.2f} per warp-node")
    for c, k in by.most_common():
        print(f"  {c:12s} {k / wn:7.2f} per warp-node   stall samples {stalls[c] / max(1, sum(stalls.values())):6.1%}")
    print("  fp64 by opcode: " + ", ".join(f"{o} {k / wn:.2f}" for o, k in fp64_ops.most_common()))
    print(f"  register-file read cycles (bank model) {rf / wn:.1f} per warp-node")
    if a.json:
        try:
            with open(a.json) as f:
                d = json.load(f)
        except (OSError, ValueError):
            d = {}
        d[a.key] = {"warp_instr_per_warp_node": round(total / wn, 3),
                    "fp64_instr_per_warp_node": round(by["fp64"] / wn, 3),
                    "per_class": {c: round(k / wn, 3) for c, k in by.items()},
                    "rf_read_cycles_per_warp_node": round(rf / wn, 2),
                    "source": f"ncu --set full source page of {a.rep.split('/')[-1]} (n = {a.n})"}
        with open(a.json, "w") as f:
            json.dump(d, f, indent=1)


if __name__ == "__main__":
    main()
