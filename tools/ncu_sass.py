"""Summarise an `ncu --page source --csv --print-source sass` dump: memory instructions with their
sector counts and the hottest instructions by stall samples. Usage: ncu_sass.py file.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr) and r[0] != 'Address']


def num(r, k):
    try:
        return float(r[ix[k]])
    except Exception:
        return 0.0


tot = sum(num(r, '# Samples') for r in data)
inst = sum(num(r, 'Instructions Executed') for r in data)
print('sass lines', len(data), 'samples', tot, 'warp insts', inst)
print('--- memory instructions')
for r in data:
    src = r[ix['Source']]
    if any(t in src for t in ('LDG', 'STG', 'ATOM', 'RED.', 'LDS', 'STS', 'LDL', 'STL')):
        print(r[ix['Address']][-5:], src[:64].ljust(64), 'ex %.3g' % num(r, 'Instructions Executed'),
              'thr %.1f' % num(r, 'Avg. Threads Executed'), 'tag %.3g' % num(r, 'L1 Tag Requests Global'),
              'l2sec %.3g' % num(r, 'L2 Theoretical Sectors Global'), 'smp %.1f%%' % (100 * num(r, '# Samples') / tot))
print('--- hottest by samples')
for r in sorted(data, key=lambda r: -num(r, '# Samples'))[:top]:
    print(r[ix['Address']][-5:], r[ix['Source']][:64].ljust(64), 'smp %.1f%%' % (100 * num(r, '# Samples') / tot),
          'ex %.3g' % num(r, 'Instructions Executed'), 'thr %.1f' % num(r, 'Avg. Threads Executed'))
