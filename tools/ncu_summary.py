"""Summarise an .ncu-rep: key raw metrics + stall samples (run here, no GPU)."""
import csv
import io
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.per_cycle_active', 'launch__registers_per_thread', 'launch__grid_size',
        'launch__block_size', 'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum',
        'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum', 'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum',
        'l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum', 'l1tex__t_requests_pipe_lsu_mem_global_op_st.sum',
        'lts__t_sectors_op_read.sum', 'lts__t_sectors_op_write.sum', 'lts__t_sector_hit_rate.pct',
        'sm__cycles_elapsed.avg']


def main(path):
    raw = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    for v in rows[2:]:
        name = v[h.index('Kernel Name')] if 'Kernel Name' in h else '?'
        print('kernel:', name[:100])
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f'  {k} = {v[i]} {units[i]}')
        stalls = []
        for i, k in enumerate(h):
            if k.startswith('smsp__pcsamp_warps_issue_stalled_') and not k.endswith('not_issued'):
                try:
                    stalls.append((float(v[i].replace(',', '')), k.replace('smsp__pcsamp_warps_issue_stalled_', '')))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1
        print('  stall samples:', ', '.join(f'{n} {100*s/tot:.0f}%' for s, n in sorted(stalls, reverse=True)[:8]))


if __name__ == '__main__':
    for p in sys.argv[1:]:
        main(p)
