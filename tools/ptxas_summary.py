"""Summarise lib/ptxas.log: registers / spills / smem per kernel instantiation."""
import re
import subprocess
import sys

log = open(sys.argv[1] if len(sys.argv) > 1 else "paper_2103_08825_b200/lib/ptxas.log").read()
cur = None
for line in log.splitlines():
    m = re.search(r"Compiling entry function '(\w+)'", line) or re.search(r"Function properties for (\w+)", line)
    if m:
        cur = m.group(1)
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        name = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip()
        name = re.sub(r"sb::Fused1DParams<[^>]*>|sb::Geom", "", name)
        print(f"{m.group(1):>4} regs  {name[:110]}")
