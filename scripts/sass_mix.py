"""Opcode histogram (weighted by warp instructions executed) and stall samples of an
`ncu --page source --csv --print-source sass` export.  usage: sass_mix.py file.csv [top]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
iS, iE, iW = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
ops, stalls, tot, tots = collections.Counter(), collections.Counter(), 0, 0
for r in rows[2:]:
    if len(r) < len(h):
        continue
    src = r[iS].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0] if op not in ("LDS", "STS") else op
    n = float(r[iE] or 0)
    w = float(r[iW] or 0)
    ops[op] += n
    stalls[op] += w
    tot += n
    tots += w
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print(f"total warp instructions {tot:.4g}, stall samples {tots:.4g}")
for op, n in ops.most_common(top):
    print(f"{op:12s} {n / tot * 100:6.2f}% of instr  {stalls[op] / max(tots, 1) * 100:6.2f}% of samples")
