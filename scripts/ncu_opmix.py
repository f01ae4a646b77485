"""Executed-instruction mix per unit from an ncu report's SASS source page."""
import csv, re, subprocess, sys, collections
rep, units = sys.argv[1], float(sys.argv[2])
kidx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
blocks = []; hdr = None
for r in rows:
    if r and r[0] == 'Kernel Name':
        blocks.append([]); continue
    if r and r[0] == 'Address':
        hdr = r; continue
    if blocks and hdr and len(r) == len(hdr):
        blocks[-1].append(r)
b = blocks[kidx]
ie = hdr.index('Instructions Executed')
op = collections.Counter(); tot = 0
for r in b:
    n = int(r[ie] or 0)
    m = re.match(r'\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)', r[1])
    o = m.group(2) if m else r[1]
    op[o] += n; tot += n
print('warp-inst total %.0f, per unit (x32 threads) %.1f' % (tot, tot * 32 / units))
for o, n in op.most_common(32):
    print('  %-10s %7.2f' % (o, n * 32 / units))
