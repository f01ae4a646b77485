"""Summarise an ncu --set full report: per kernel the headline metrics."""
import csv, subprocess, sys
rep = sys.argv[1]
cells = float(sys.argv[2]) if len(sys.argv) > 2 else None
out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'launch__registers_per_thread',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'smsp__sass_inst_executed_op_local_ld.sum']
stalls = [h for h in hdr if h.startswith('smsp__pcsamp_warps_issue_stalled_') and not h.endswith('not_issued')]
for r in rows[2:]:
    d = dict(zip(hdr, r)); u = dict(zip(hdr, units))
    print(d['Kernel Name'][:100])
    for w in want:
        if w in d:
            extra = ''
            if cells and w == 'smsp__inst_executed.sum':
                extra = '  (%.1f thread-inst per cell)' % (float(d[w].replace(',', '')) * 32 / cells)
            print('   %-62s %s %s%s' % (w, d[w], u[w], extra))
    tot = sum(float(d[h]) for h in stalls if d[h])
    top = sorted(((float(d[h]), h) for h in stalls if d[h]), reverse=True)[:7]
    print('   stalls:', ', '.join('%s %.0f%%' % (h.replace('smsp__pcsamp_warps_issue_stalled_', ''), 100 * v / tot) for v, h in top))
