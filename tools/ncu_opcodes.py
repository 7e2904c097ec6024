"""Instruction mix and stall reasons per SASS opcode from an ncu report's
source page (needs a capture with --import-source / SourceCounters):

    ncu -i rep.ncu-rep --page source --csv --print-source sass > src.csv
    python tools/ncu_opcodes.py src.csv
"""
import csv, collections, re, sys
rows = list(csv.reader(open(sys.argv[1])))
head = rows[1]
idx = {h: i for i, h in enumerate(head)}
stalls = [h for h in head if h.startswith("stall_") and "Not Issued" not in h]
by_op = collections.defaultdict(lambda: collections.Counter())
exe = collections.Counter()
tot = collections.Counter()
for r in rows[2:]:
    if len(r) < len(head): continue
    src = r[idx["Source"]].strip()
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", src)
    if not m: continue
    op = m.group(2)
    ie = int(r[idx["Instructions Executed"]] or 0)
    exe[op] += ie
    for s in stalls:
        v = int(r[idx[s]] or 0)
        by_op[op][s] += v
        tot[s] += v
T = sum(exe.values())
print("executed instructions by opcode (top 15):")
for op, c in exe.most_common(15):
    print(f"  {op:10s} {c:14d} {100*c/T:5.1f}%   stalls: " + ", ".join(f"{k[6:]}={v}" for k, v in by_op[op].most_common(4)))
S = sum(tot.values())
print("stall totals:", ", ".join(f"{k[6:]} {100*v/S:.0f}%" for k, v in tot.most_common(10)))
