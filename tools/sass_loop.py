"""Dump a kernel's SASS with stall counts from a built .so (experiment helper).

    python tools/sass_loop.py LIB.so NAME_SUBSTRING [start_hex end_hex]
"""
import re
import subprocess
import sys

lib, sub = sys.argv[1], sys.argv[2]
rng = (int(sys.argv[3], 16), int(sys.argv[4], 16)) if len(sys.argv) > 4 else None
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
for p in re.split(r"\n\s*Function : ", txt)[1:]:
    name = p.split("\n")[0]
    if sub not in name:
        continue
    lines = p.split("\n")
    i = 0
    while i < len(lines):
        m = re.match(r"\s+/\*([0-9a-f]{4,5})\*/\s+(.*?);\s+/\* (0x[0-9a-f]+) \*/", lines[i])
        if m and i + 1 < len(lines):
            m2 = re.match(r"\s+/\* (0x[0-9a-f]+) \*/", lines[i + 1])
            if m2:
                word = int(m.group(3), 16) | (int(m2.group(1), 16) << 64)
                addr = int(m.group(1), 16)
                if rng is None or rng[0] <= addr <= rng[1]:
                    print(f"{addr:05x} st={(word >> 105) & 0xf:2d} {m.group(2).strip()}")
                i += 2
                continue
        i += 1
    break
