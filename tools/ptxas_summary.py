"""Summarise ptxas -v output (registers / spills / smem per kernel) from build/*.ptxas.txt."""
import glob
import os
import re
import subprocess
import sys

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for f in sorted(glob.glob(os.path.join(root, "paper_2005_06727_b200", "build", "*.ptxas.txt"))):
    txt = open(f).read().splitlines()
    name = None
    spill = ""
    for line in txt:
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
            name = re.sub(r"wmd::\(anonymous namespace\)::", "", name)
            name = re.sub(r"\(.*", "", name)
        m = re.search(r"(\d+) bytes spill stores", line)
        if m:
            spill = m.group(1)
        m = re.search(r"Used (\d+) registers", line)
        if m and name:
            print(f"{name:60s} regs={m.group(1):>4} spill={spill:>4} {line.split('barriers')[-1].strip(', ')}")
            name = None
