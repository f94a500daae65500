"""Executed instructions / stall samples of a stage kernel grouped by kernel phase
(outermost tp_kernels.cu line of the inline chain).  usage: ncu_phases.py rep.ncu-rep '(bool)1, (bool)0' lib.so"""
import csv, collections, re, subprocess, sys, tempfile, os, glob
rep, ksub, so = sys.argv[1], sys.argv[2], os.path.abspath(sys.argv[3])
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=tmp, capture_output=True)
cub = [c for c in glob.glob(tmp + "/*.cubin") if "tp_kernels" in c][0]
dis = subprocess.run(["nvdisasm", "-gi", "-c", cub], capture_output=True, text=True).stdout.split("\n")
src = open(os.environ.get("TP_KSRC", "/root/repo/paper_2104_06784_b200/csrc/tp_kernels.cu")).read().split("\n")
func = None; cur = None; mp = collections.defaultdict(dict)
for ln in dis:
    m = re.match(r'\s*\.text\.(\S+):', ln)
    if m: func = m.group(1); continue
    if "//## File" in ln:
        locs = re.findall(r'"([^"]+)", line (\d+)', ln)
        outer = [int(l) for f, l in locs if f.endswith("tp_kernels.cu")]
        cur = outer[-1] if outer else None
        continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', ln)
    if m and func: mp[func][int(m.group(1), 16)] = cur
# phase boundaries from markers in the source
marks = {}
for i, l in enumerate(src, 1):
    for key in ("// ---- Phase 1:", "// ---- Phase 2:", "// ---- Phase 3:", "// ---- boundary mass tally"):
        if key in l and key not in marks:
            marks[key.replace("// ---- ", "")] = i
start_kernel = [i for i, l in enumerate(src, 1) if "__global__ void __launch_bounds__(NT, 2) stage_kernel" in l][0]
def phase(line):
    if line is None: return "?"
    if line < start_kernel: return "epilogue/helpers"
    if line < marks["Phase 1:"]: return "prologue/TMA"
    if line < marks["Phase 2:"]: return "phase1 faces+cells"
    if line < marks["Phase 3:"]: return "phase2 brackets"
    if line < marks["boundary mass tally"]: return "phase3 sources/update"
    return "tally/loop"
page = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout.split("\n")
blocks = []; curb = None
for ln in page:
    if ln.startswith('"Kernel Name"'):
        curb = [ln]; blocks.append(curb)
    elif curb is not None:
        curb.append(ln)
for b in blocks:
    if ksub not in b[0]: continue
    rows = list(csv.reader(b[1:])); hdr = rows[0]; data = [r for r in rows[1:] if len(r) == len(hdr)]
    si = hdr.index("Warp Stall Sampling (All Samples)"); ii = hdr.index("Instructions Executed")
    m = re.search(r'\(bool\)(\d), \(bool\)(\d)', b[0])
    fname = [f for f in mp if "stage_kernel" in f and f"ILb{m.group(1)}ELb{m.group(2)}E" in f][0]
    base = int(data[0][0], 16)
    S = collections.Counter(); I = collections.Counter(); OPS = collections.defaultdict(collections.Counter)
    for r in data:
        ph = phase(mp[fname].get(int(r[0], 16) - base))
        S[ph] += int(r[si]); I[ph] += int(r[ii])
        op = r[1].strip().split(); op = (op[1] if op[0].startswith('@') else op[0]).split('.')[0]
        OPS[ph][op] += int(r[ii])
    ts, ti = sum(S.values()), sum(I.values())
    print(b[0][:80], f"total insts {ti/1e6:.1f}M")
    for ph in sorted(I, key=lambda p: -I[p]):
        top = ", ".join(f"{o} {100*v/I[ph]:.0f}%" for o, v in OPS[ph].most_common(6))
        print(f"  {ph:24s} insts {100*I[ph]/ti:5.1f}%  samples {100*S[ph]/ts:5.1f}%   [{top}]")
    break
