"""Summarise an ncu report: key metrics per kernel launch (used for profiles/)."""
import csv, subprocess, sys

SECTIONS = ('GPU Speed Of Light Throughput', 'Memory Workload Analysis', 'Compute Workload Analysis',
            'Scheduler Statistics', 'Warp State Statistics', 'Occupancy', 'Launch Statistics')
KEEP = ('Duration', 'DRAM Throughput', 'Memory Throughput', 'L1/TEX Hit Rate', 'L2 Hit Rate',
        'Compute (SM) Throughput', 'Executed Ipc Active', 'Issue Slots Busy', 'No Eligible',
        'Eligible Warps Per Scheduler', 'Warp Cycles Per Issued Instruction',
        'Avg. Active Threads Per Warp', 'Achieved Occupancy', 'Theoretical Occupancy',
        'Registers Per Thread', 'Grid Size', 'Block Size', 'Dynamic Shared Memory Per Block',
        'Block Limit Shared Mem', 'Block Limit Registers', 'Mem Busy', 'Max Bandwidth',
        'L1/TEX Cache Throughput', 'L2 Cache Throughput')


def main(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[0]
    ki, si, mi, vi, ui, idi = (h.index(k) for k in ('Kernel Name', 'Section Name', 'Metric Name',
                                                      'Metric Value', 'Metric Unit', 'ID'))
    cur = None
    for x in r[1:]:
        if x[idi] != cur:
            cur = x[idi]
            print('\n== launch %s: %s' % (cur, x[ki][:90]))
        if x[si] in SECTIONS and x[mi] in KEEP:
            print('   %-40s %s %s' % (x[mi], x[vi], x[ui]))
    raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) > 2:
        hh = rr[0]
        want = [i for i, n in enumerate(hh) if n in (
            'dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__time_duration.sum',
            'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
            'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
            'smsp__inst_executed.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active',
            'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum',
            'lts__t_sectors_srcunit_tex_op_read.sum')]
        print('\nraw:')
        for row in rr[2:]:
            print('  ', rr[0][0], row[0], {hh[i]: row[i] + ' ' + rr[1][i] for i in want})


if __name__ == '__main__':
    main(sys.argv[1])
