"""Per-source-line stall breakdown from an ncu source-page CSV (tools/gpu_ncu_src.sh).
usage: python tools/sass_stalls.py page.csv cubin kernel_substring [file:lo-hi ...]"""
import csv, io, re, subprocess, sys
from collections import defaultdict
page, cubin, kname = sys.argv[1:4]
rows = list(csv.reader(open(page)))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
base = min(int(d['Address'], 16) for d in data)
dis = subprocess.run(['nvdisasm', '-g', '-c', cubin], capture_output=True, text=True).stdout
off2line, cur, line = {}, None, None
for l in dis.splitlines():
    m = re.match(r'\s*\.text\.(\S+):', l)
    if m: cur = m.group(1); continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m: line = (m.group(1).split('/')[-1], int(m.group(2))); continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', l)
    if m and cur and kname in cur: off2line[int(m.group(1), 16)] = line
keys = [k for k in hdr if k.startswith('stall_') and 'Not Issued' not in k]
agg = defaultdict(lambda: defaultdict(int)); tot = 0
for d in data:
    ln = off2line.get(int(d['Address'], 16) - base)
    s = int(d['Warp Stall Sampling (All Samples)']); tot += s
    agg[ln]['all'] += s
    for k in keys: agg[ln][k] += int(d[k] or 0)
def show(title, sel):
    a = defaultdict(int)
    for ln, v in agg.items():
        if sel(ln):
            for k, x in v.items(): a[k] += x
    top = sorted(((a[k], k) for k in keys), reverse=True)[:6]
    print(f"{title}: {100*a['all']/tot:5.1f}% of samples; " + ", ".join(f"{k[6:]} {100*x/max(a['all'],1):.0f}%" for x, k in top))
for spec in sys.argv[4:]:
    f, r = spec.split(':'); lo, hi = (int(x) for x in r.split('-'))
    show(spec, lambda ln: ln and ln[0] == f and lo <= ln[1] <= hi)
for ln, v in sorted(agg.items(), key=lambda kv: -kv[1]['all'])[:30]:
    top = sorted(((v[k], k) for k in keys), reverse=True)[:3]
    print(f"{100*v['all']/tot:5.1f}% {str(ln):30s} " + ", ".join(f"{k[6:]} {x}" for x, k in top))
