"""Top stalled SASS instructions of an ncu report (source page)."""
import csv, subprocess, sys
rep = sys.argv[1]; kidx = int(sys.argv[2]) if len(sys.argv) > 2 else 0; top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
blocks = []; hdr = None
for r in rows:
    if r and r[0] == 'Kernel Name': blocks.append([]); continue
    if r and r[0] == 'Address': hdr = r; continue
    if blocks and hdr and len(r) == len(hdr): blocks[-1].append(r)
b = blocks[kidx]
si = hdr.index('Warp Stall Sampling (All Samples)')
cols = [c for c in hdr if c.startswith('stall_') and '(Not Issued)' not in c]
tot = sum(float(r[si] or 0) for r in b)
rank = sorted(b, key=lambda r: -float(r[si] or 0))[:top]
for r in rank:
    st = sorted(((float(r[hdr.index(c)] or 0), c) for c in cols), reverse=True)[:2]
    print('%5.1f%% %-60s %s' % (100 * float(r[si] or 0) / tot, r[1].strip()[:60], ' '.join('%s:%.0f' % (c[6:], v) for v, c in st)))
