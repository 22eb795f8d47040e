"""Spill summary per K2 instantiation from `nvcc -Xptxas -v` output on stdin."""
import re
import sys

cur = None
for line in sys.stdin:
    m = re.search(r"Function properties for (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur and "spmm_sm100_kernel" in cur:
        nh = re.search(r"spmm_sm100_kernelILi(\d+)E", cur).group(1)
        teams = re.search(r"TeamsILi(\d)ELi(\d)ELi(\d)ELi(\d+)E((?:Lb[01]E)+)", cur)
        flags = re.findall(r"Lb([01])E", teams.group(5))
        iss = re.search(r"EEELi(\d)EEEv", cur)
        print("NH=%s T=%s W=%s KG=%s flags=%s I=%s" % (nh, teams.group(1), teams.group(2), teams.group(4),
                                                       "".join(flags), iss.group(1) if iss else "?"),
              "stack", m.group(1), "spill st/ld", m.group(2), m.group(3))
        cur = None
