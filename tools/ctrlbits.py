"""Decode Volta+ SASS control bits (stall/yield/wbar/rbar/wait-mask) from cuobjdump -sass output."""
import re, sys
lines = sys.stdin.read().splitlines()
i = 0
out = []
while i < len(lines):
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);\s*/\* (0x[0-9a-f]+) \*/", lines[i])
    if m and i + 1 < len(lines):
        m2 = re.search(r"/\* (0x[0-9a-f]+) \*/", lines[i + 1])
        if m2:
            hi = int(m2.group(1), 16)
            ctrl = hi >> 41  # bits 105.. of the 128-bit word
            stall = ctrl & 0xF; yld = (ctrl >> 4) & 1; wbar = (ctrl >> 5) & 7; rbar = (ctrl >> 8) & 7
            wait = (ctrl >> 11) & 0x3F
            out.append(f"{m.group(1)} {m.group(2)[:60]:60s} st={stall:2d} y={yld} wb={wbar} rb={rbar} wait={wait:06b}")
            i += 2
            continue
    i += 1
print("\n".join(out))
