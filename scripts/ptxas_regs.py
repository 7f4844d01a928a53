"""Registers / spills per kernel from the ptxas logs the build writes
(paper_1705_01167_b200/build/*.ptxas.log). Usage: python scripts/ptxas_regs.py [filter]"""
import re
import subprocess
import sys
from pathlib import Path

LOGS = Path(__file__).resolve().parents[1] / "paper_1705_01167_b200" / "build"
pat = sys.argv[1] if len(sys.argv) > 1 else ""
for log in sorted(LOGS.glob("*.ptxas.log")):
    fn = None
    spill = ""
    for line in log.read_text().splitlines():
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            fn = m.group(1)
            continue
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m:
            spill = f"spill {m.group(1)}/{m.group(2)}"
        m = re.search(r"Used (\d+) registers", line)
        if m and fn:
            name = subprocess.run(["c++filt", fn], capture_output=True, text=True).stdout.strip()
            if pat in name and "cub::" not in name:
                print(f"{m.group(1):>4} regs {spill:>16}  {name[:150]}")
            fn, spill = None, ""
