"""Attribute ncu per-SASS-instruction stall samples to CUDA source lines.
usage: python tools/sass_lines.py report.ncu-rep kernel_substring cubin"""
import csv, io, re, subprocess, sys
from collections import defaultdict
rep, kname, cubin = sys.argv[1:4]
txt = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
base = min(int(d['Address'], 16) for d in data)
# line info from nvdisasm
dis = subprocess.run(['nvdisasm', '-g', '-c', cubin], capture_output=True, text=True).stdout
func = None; line = None; off2line = {}
cur_func = None
for l in dis.splitlines():
    m = re.match(r'\s*\.text\.(\S+):', l)
    if m: cur_func = m.group(1); continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m: line = (m.group(1).split('/')[-1], int(m.group(2))); continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', l)
    if m and cur_func and kname in cur_func:
        off2line[int(m.group(1), 16)] = line
agg = defaultdict(lambda: [0, 0]); tot = 0
for d in data:
    off = int(d['Address'], 16) - base
    ln = off2line.get(off)
    s = int(d['Warp Stall Sampling (All Samples)']); tot += s
    agg[ln][0] += s; agg[ln][1] += int(d['Instructions Executed'])
srcs = {}
for (ln, (s, i)) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:45]:
    src = ''
    if ln:
        fn = {'btd_small.cuh': 'paper_2509_03015_b200/csrc/btd_small.cuh', 'btd_factor.cuh': 'paper_2509_03015_b200/csrc/btd_factor.cuh', 'btd_solve.cuh': 'paper_2509_03015_b200/csrc/btd_solve.cuh', 'btd_device.cuh': 'paper_2509_03015_b200/csrc/btd_device.cuh'}.get(ln[0])
        if fn:
            src = open(fn).read().splitlines()[ln[1] - 1].strip()[:70]
    print(f"{100*s/tot:5.1f}%  inst {i:11d}  {str(ln):32s} {src}")
