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
        t = re.search(r"spmm_sm100_kernelILi(\d+)ENS0_5TeamsILi(\d)ELi(\d)ELi(\d)ELi(\d+)ELb([01])EEELi(\d)", cur)
        print("NH=%s T=%s W=%s KG=%s ZF=%s I=%s" % (t.group(1), t.group(2), t.group(3), t.group(5), t.group(6), t.group(7)),
              "stack", m.group(1), "spill st/ld", m.group(2), m.group(3))
        cur = None
