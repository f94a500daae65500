"""Stall samples / executed instructions per source line for one kernel of an ncu report.
usage: ncu_lines.py report.ncu-rep <kernel-substring> <so-file> [topN]"""
import csv, collections, re, subprocess, sys, tempfile, os, glob
rep, ksub, so = sys.argv[1], sys.argv[2], os.path.abspath(sys.argv[3])
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=tmp, capture_output=True)
cub = [c for c in glob.glob(tmp + "/*.cubin") if os.path.getsize(c) > 100000][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout.split("\n")
func = None; cur = None; mp = collections.defaultdict(dict)
for ln in dis:
    m = re.match(r'\s*\.text\.(\S+):', ln)
    if m: func = m.group(1); continue
    m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', ln)
    if m: cur = (m.group(1), int(m.group(2))); continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', ln)
    if m and func: mp[func][int(m.group(1), 16)] = cur
page = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout.split("\n")
blocks = []; curb = None
for ln in page:
    if ln.startswith('"Kernel Name"'):
        curb = [ln]; blocks.append(curb)
    elif curb is not None:
        curb.append(ln)
for b in blocks:
    if ksub not in b[0]:
        continue
    kname = b[0]
    rows = list(csv.reader(b[1:])); hdr = rows[0]; data = [r for r in rows[1:] if len(r) == len(hdr)]
    si = hdr.index("Warp Stall Sampling (All Samples)"); ii = hdr.index("Instructions Executed")
    # find mangled name with the same SASS length
    m = re.search(r'\(bool\)(\d), \(bool\)(\d)', kname)
    cands = [f for f in mp if 'stage_kernel' in f and (not m or f'ILb{m.group(1)}ELb{m.group(2)}E' in f)]
    base = int(data[0][0], 16)
    nins = len(data)
    fname = min(cands, key=lambda f: abs(len(mp[f]) - nins))
    agg = collections.Counter(); aggi = collections.Counter(); op_s = collections.Counter(); op_i = collections.Counter()
    for r in data:
        key = mp[fname].get(int(r[0], 16) - base)
        agg[key] += int(r[si]); aggi[key] += int(r[ii])
        op = r[1].strip().split()
        op = (op[1] if op[0].startswith('@') else op[0]).split('.')[0]
        op_s[op] += int(r[si]); op_i[op] += int(r[ii])
    tot = sum(agg.values()); toti = sum(aggi.values())
    print(kname[:90], "samples", tot, "insts", toti, "matched", fname[:50])
    srcs = {}
    for key, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
        line = ""
        if key:
            path = glob.glob(f"/root/repo/paper_2104_06784_b200/csrc/{key[0]}")
            if path:
                srcs.setdefault(key[0], open(path[0]).read().split("\n"))
                line = srcs[key[0]][key[1] - 1].strip()[:70]
        print(f"  {str(key):32s} {100*v/tot:5.1f}% smp {100*aggi[key]/toti:5.1f}% ins | {line}")
    print("  by opcode:", ", ".join(f"{k} {100*v/toti:.1f}%i/{100*op_s[k]/tot:.1f}%s" for k, v in op_i.most_common(16)))
    break
