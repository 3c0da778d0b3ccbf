"""Key metrics of an ncu --set full report: python tools/ncu_summary.py rep.ncu-rep"""
import csv, subprocess, sys, io
WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sector_hit_rate.pct',
        'lts__t_bytes.sum', 'l1tex__t_sector_hit_rate.pct',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__thread_inst_executed_per_inst_executed.ratio',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__grid_size', 'launch__block_size',
        'launch__registers_per_thread', 'smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_membar_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio']
for path in sys.argv[1:]:
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u = r[0], r[1]
    print('==', path)
    for row in r[2:]:
        name = row[h.index('Kernel Name')] if 'Kernel Name' in h else ''
        print('kernel:', name[:80])
        for w in WANT:
            if w in h:
                i = h.index(w)
                print(f'  {w:78s} {row[i]:>18s} {u[i]}')
        # every other warp-stall reason above 0.5 per issue, plus instruction / shared-memory counts
        for i, w in enumerate(h):
            if w in WANT:
                continue
            ok = ('issue_stalled' in w and w.endswith('per_issue_active.ratio')) or w in (
                'smsp__inst_executed.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
                'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum', 'l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum',
                'sm__warps_active.avg.per_cycle_active', 'launch__occupancy_limit_registers',
                'launch__occupancy_limit_shared_mem', 'sm__maximum_warps_per_active_cycle_pct')
            if not ok:
                continue
            try:
                v = float(row[i].replace(',', ''))
            except ValueError:
                continue
            if 'issue_stalled' in w and v < 0.5:
                continue
            print(f'  {w:78s} {row[i]:>18s} {u[i]}')
