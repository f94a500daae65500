"""Per-source-line executed instructions and stall samples of one stage kernel from an ncu
report (SASS page) mapped through nvdisasm line info of the built library (development aid).
usage: ncu_lines2.py rep.ncu-rep '(bool)1, (bool)1' lib.so [outer|inner] [N]"""
import csv, collections, re, subprocess, sys, tempfile, os, glob
rep, ksub, so = sys.argv[1], sys.argv[2], os.path.abspath(sys.argv[3])
mode = sys.argv[4] if len(sys.argv) > 4 else "outer"
N = int(sys.argv[5]) if len(sys.argv) > 5 else 40
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=tmp, capture_output=True)
cub = [c for c in glob.glob(tmp + "/*.cubin") if "tp_kernels" in c][0]
dis = subprocess.run(["nvdisasm", "-gi", "-c", cub], capture_output=True, text=True).stdout.split("\n")
func = None; chain = []; fresh = True; mp = collections.defaultdict(dict)
for ln in dis:
    m = re.match(r'\s*\.text\.(\S+):', ln)
    if m: func = m.group(1); continue
    if "//## File" in ln:
        if fresh:
            chain = []; fresh = False
        chain.extend(re.findall(r'"([^"]+)", line (\d+)', ln))
        continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', ln)
    if m and func:
        fresh = True
        if chain:
            if mode == "outer":   # the stage_kernel body line (last tp_kernels.cu line before the kernel's own)
                ks = [(f, l) for f, l in chain if f.endswith("tp_kernels.cu")]
                f, l = ks[-2] if len(ks) > 1 else ks[-1] if ks else chain[-1]
            elif mode == "mid":   # the innermost tp_kernels.cu line
                ks = [(f, l) for f, l in chain if f.endswith("tp_kernels.cu")]
                f, l = ks[0] if ks else chain[0]
            else:
                f, l = chain[0]
            mp[func][int(m.group(1), 16)] = (os.path.basename(f), int(l))
page = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout.split("\n")
blocks = []; curb = None
for ln in page:
    if ln.startswith('"Kernel Name"'):
        curb = [ln]; blocks.append(curb)
    elif curb is not None:
        curb.append(ln)
srcs = {}
def srcline(f, l):
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2104_06784_b200", "csrc", f)
    if p not in srcs:
        srcs[p] = open(p).read().split("\n") if os.path.exists(p) else []
    s = srcs[p]
    return s[l - 1].strip()[:70] if 0 < l <= len(s) else ""
for b in blocks:
    if ksub not in b[0]: continue
    rows = list(csv.reader(b[1:])); hdr = rows[0]; data = [r for r in rows[1:] if len(r) == len(hdr)]
    si = hdr.index("Warp Stall Sampling (All Samples)"); ii = hdr.index("Instructions Executed")
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    # the exact instance: every template argument (FD, CORR, PEER, NTH) of the reported kernel
    m = re.search(r'\(bool\)(\d), \(bool\)(\d), \(bool\)(\d), \(int\)(\d+)', b[0])
    key = f"ILb{m.group(1)}ELb{m.group(2)}ELb{m.group(3)}ELi{m.group(4)}E"
    fname = [f for f in mp if "stage_kernel" in f and key in f][0]
    base = int(data[0][0], 16)
    S = collections.Counter(); I = collections.Counter(); R = collections.defaultdict(collections.Counter)
    for r in data:
        loc = mp[fname].get(int(r[0], 16) - base)
        S[loc] += int(r[si]); I[loc] += int(r[ii])
        for h in reasons:
            R[loc][h] += int(r[hdr.index(h)] or 0)
    ts, ti = sum(S.values()), sum(I.values())
    print(b[0][:80], f"total insts {ti/1e6:.1f}M samples {ts}")
    for loc in sorted(S, key=lambda p: -S[p])[:N]:
        top = ",".join(f"{h[6:]}{100*v/max(S[loc],1):.0f}" for h, v in R[loc].most_common(3))
        f, l = loc if loc else ("?", 0)
        print(f"  {f}:{l:<5d} smp {100*S[loc]/ts:5.1f}% ins {100*I[loc]/ti:5.1f}%  [{top}]  {srcline(f, l)}")
    break
