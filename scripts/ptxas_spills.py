"""Summarise ptxas -v output: registers / spill bytes per kernel instantiation."""
import re
import sys

txt = open(sys.argv[1]).read()
cur = None
for line in txt.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        name = m.group(1)
        t = re.search(r"(match_tc_kernel|[a-z_]+_kernel)I(.*?)EE", name)
        cur = (t.group(1) + "<" + ",".join(re.findall(r"Li(\d+)E", t.group(2))) + ">") if t else name[-60:]
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        st, ld = m.groups()
        if len(sys.argv) < 3 or sys.argv[2] in cur:
            print(f"{cur:40s} spill st {st:>5s} ld {ld:>5s}")
        cur = None
