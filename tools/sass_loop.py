"""Dev tool: SASS audit of a kernel's hot loop.

    python tools/sass_loop.py lib.so <function-substring> [--dump]

Extracts the function from `cuobjdump -sass`, finds the innermost backward
branch whose body contains LDS (the leaf loop that reads the TMA ring) and
prints the opcode histogram of that body (instructions per iteration)."""
import collections
import re
import subprocess
import sys


def functions(lib):
    """Yield (name, [(addr, text, ctrl)]) with ctrl = decoded control bits of
    the instruction's high word: stall [105:109), yield, wbar, rbar,
    wait_mask [116:122), reuse [122:126)."""
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    cur, body = None, []
    lines = out.split("\n")
    for i, line in enumerate(lines):
        m = re.search(r"Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,6})\*/\s+(.*?);", line)
        if m and cur:
            hm = re.search(r"/\* (0x[0-9a-f]{16}) \*/", lines[i + 1]) if i + 1 < len(lines) else None
            hi = int(hm.group(1), 16) if hm else 0
            ctrl = dict(stall=(hi >> 41) & 0xF, yld=(hi >> 45) & 1, wbar=(hi >> 46) & 7, rbar=(hi >> 49) & 7,
                        wait=(hi >> 52) & 0x3F, reuse=(hi >> 58) & 0xF)
            body.append((int(m.group(1), 16), m.group(2).strip(), ctrl))
    if cur:
        yield cur, body


def main():
    import signal; signal.signal(signal.SIGPIPE, signal.SIG_DFL)
    lib, pat = sys.argv[1], sys.argv[2]
    for name, ins in functions(lib):
        if pat not in name:
            continue
        loops = []
        for a, t, _ in ins:
            m = re.search(r"BRA\S*\s+.*?(0x[0-9a-f]+)\s*$", t)
            if m and int(m.group(1), 16) < a:
                lo, hi = int(m.group(1), 16), a
                body = [x for x in ins if lo <= x[0] <= hi]
                # the leaf loop reads the ring with vector LDS (.64/.128);
                # short spin loops on a shared-memory word do not count
                if any(re.search(r"\bLDS\.(64|128)", x[1]) for x in body):
                    loops.append((hi - lo, lo, hi, body))
        if not loops:
            print(name, "no LDS loop")
            continue
        _, lo, hi, body = min(loops)
        c = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0] for _, t, _ in body)
        stall = sum(x[2]["stall"] for x in body)
        reuse = sum(bin(x[2]["reuse"]).count("1") for x in body)
        print(f"{name}: loop {hex(lo)}..{hex(hi)}: {len(body)} instructions, "
              f"sum of stall fields {stall} cycles, {reuse} reuse flags")
        for k, v in c.most_common():
            print(f"  {v:5d} {k}")
        if "--dump" in sys.argv:
            for a, t, c in body:
                print(f"    {a:05x} s{c['stall']:<2d} {'R' * bin(c['reuse']).count('1'):3s} {t}")


if __name__ == "__main__":
    main()
