"""Dynamic opcode mix (warp instructions executed, thread instructions, stall samples) of each
kernel in an ncu SASS source-page CSV export (development aid):
  ncu -i rep --page source --csv --print-source sass > x.csv; python ncu_opmix.py x.csv"""
import csv, collections, re, sys
blocks = []; cur = None
for ln in open(sys.argv[1]):
    if ln.startswith('"Kernel Name"'):
        cur = [ln]; blocks.append(cur)
    elif cur is not None:
        cur.append(ln)
for b in blocks:
    rows = list(csv.reader(b[1:])); hdr = rows[0]; data = [r for r in rows[1:] if len(r) == len(hdr)]
    ii = hdr.index("Instructions Executed"); ti = hdr.index("Thread Instructions Executed")
    si = hdr.index("Warp Stall Sampling (All Samples)")
    I = collections.Counter(); T = collections.Counter(); S = collections.Counter()
    for r in data:
        src = r[1].strip()
        src = re.sub(r'^@!?U?P\w+\s+', '', src)
        op = src.split(' ')[0].split('.')[0] if src else '?'
        I[op] += int(r[ii]); T[op] += int(r[ti]); S[op] += int(r[si])
    ti_ = sum(I.values()); ts = sum(S.values())
    print(b[0].split(',')[1][:90], f"warp insts {ti_/1e6:.1f}M")
    for op, v in I.most_common(32):
        print(f"  {op:10s} {100*v/ti_:5.1f}% inst  thr/warp {T[op]/max(v,1):5.1f}  {100*S[op]/ts:5.1f}% samples")
