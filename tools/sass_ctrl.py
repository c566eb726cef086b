"""Decode Volta+ SASS control bits (stall, yield, write/read scoreboard,
wait mask) from `cuobjdump -sass` output, to see how loads are assigned to
the 6 dependency scoreboards and where the warp waits on them."""
import re
import sys


def parse(text):
    lines = text.splitlines()
    out = []
    i = 0
    while i < len(lines):
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);\s+/\* (0x[0-9a-f]+) \*/", lines[i])
        if m and i + 1 < len(lines):
            m2 = re.match(r"\s+/\* (0x[0-9a-f]+) \*/", lines[i + 1])
            if m2:
                hi = int(m2.group(1), 16)
                ctrl = hi >> 41
                stall = ctrl & 0xF
                yld = (ctrl >> 4) & 1
                wb = (ctrl >> 5) & 7
                rb = (ctrl >> 8) & 7
                wait = (ctrl >> 11) & 0x3F
                out.append((m.group(1), m.group(2).strip(), stall, yld, wb, rb, wait))
                i += 2
                continue
        i += 1
    return out


if __name__ == "__main__":
    text = open(sys.argv[1]).read()
    lo, hi = (int(sys.argv[2], 16), int(sys.argv[3], 16)) if len(sys.argv) > 3 else (0, 1 << 40)
    for addr, ins, stall, yld, wb, rb, wait in parse(text):
        a = int(addr, 16)
        if lo <= a <= hi:
            w = "".join(str(b) for b in range(6) if wait >> b & 1)
            print(f"{addr} S{stall:02d} {'Y' if yld else ' '} wb{wb if wb != 7 else '-'} rb{rb if rb != 7 else '-'} "
                  f"wait[{w:6s}] {ins}")
