"""Per-function SASS statistics of libgmres.so (dev tool): local-memory ops, barriers, TMA."""
import re, subprocess, sys
lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2011_01850_b200/libgmres.so"
pat = sys.argv[2] if len(sys.argv) > 2 else "solve_kernel"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
cur, stats = None, {}
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1); stats[cur] = {}
        continue
    if cur is None: continue
    m = re.search(r"/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
    if m:
        op = m.group(2).split(".")[0]
        stats[cur][op] = stats[cur].get(op, 0) + 1
for f, s in stats.items():
    if pat in f:
        keys = ["LDL", "STL", "MEMBAR", "CCTL", "UBLKCP", "SYNCS", "BAR", "LDG", "STG", "RED", "ATOMG"]
        print(f[:70], " ".join(f"{k}={s.get(k,0)}" for k in keys), "total", sum(s.values()))
