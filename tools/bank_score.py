"""Dev tool: static register-bank score of a kernel's hot loop (the bank model
of DESIGN.md §8): per instruction, the distinct source registers read from the
even and from the odd bank (a double operand Rk reads Rk and Rk+1; operands
flagged .reuse come from the operand cache), cost = max(pipe cycles, reads of
the busier bank) with 2 pipe cycles for FP64 instructions and 1 otherwise.

    python tools/bank_score.py lib.so <function-substring> [...]"""
import re
import sys

sys.path.insert(0, "tools")
from sass_loop import functions  # noqa: E402

FP64 = ("DFMA", "DMUL", "DADD", "DSETP")


def score(body):
    total = 0
    for _, text, ctrl in body:
        parts = text.split()
        if not parts:
            continue
        i = 1 if parts[0].startswith("@") else 0
        op = parts[i]
        args = " ".join(parts[i + 1:])
        srcs = args.split(",")[1:] if "," in args else []
        wide = op.startswith(FP64)
        even, odd = set(), set()
        for sidx, a in enumerate(srcs):
            for m in re.finditer(r"\bR(\d+)(\.reuse)?", a):
                if m.group(2):
                    continue
                r = int(m.group(1))
                if wide:
                    even.add(r & ~1)
                    odd.add(r | 1)
                elif r % 2 == 0:
                    even.add(r)
                else:
                    odd.add(r)
        total += max(2 if wide else 1, len(even), len(odd))
    return total


def main():
    lib = sys.argv[1]
    for pat in sys.argv[2:]:
        for name, ins in functions(lib):
            if pat not in name:
                continue
            loops = []
            for a, t, _ in ins:
                m = re.search(r"BRA\S*\s+.*?(0x[0-9a-f]+)\s*$", t)
                if m and int(m.group(1), 16) < a:
                    lo = int(m.group(1), 16)
                    body = [x for x in ins if lo <= x[0] <= a]
                    if any(re.search(r"\bLDS\.(64|128)", x[1]) for x in body):
                        loops.append(body)
            if not loops:
                continue
            body = min(loops, key=len)
            print(f"{lib} {name[:60]}: {len(body)} instr, bank score {score(body)} cycles")
            break


if __name__ == "__main__":
    main()
