"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv, sys
from collections import OrderedDict
for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    hdr = rows[0]
    iname, ival, iunit = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
    scale = {'nsecond': 1e-3, 'usecond': 1.0, 'msecond': 1e3, 'ns': 1e-3, 'us': 1.0, 'ms': 1e3}
    tot = 0.0
    print(f)
    for r in rows[1:]:
        us = float(r[ival].replace(',', '')) * scale.get(r[iunit], 1.0)
        tot += us
        print(f"  {r[iname][:60]:60s} {us:10.1f} us")
    print(f"  {'TOTAL':60s} {tot:10.1f} us")
