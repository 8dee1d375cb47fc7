"""Print key metrics and stall reasons of an ncu report: python tools/ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__grid_size', 'launch__block_size', 'smsp__inst_executed.sum', 'lts__t_bytes.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'launch__shared_mem_per_block_dynamic', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'sm__cycles_elapsed.avg.per_second']


def main(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        print('kernel:', v[h.index('Kernel Name')][:90] if 'Kernel Name' in h else '?')
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f'  {k:66s} {v[i]:>18s} {u[i]}')
        st = [(h[i], v[i]) for i in range(len(h)) if h[i].startswith('smsp__pcsamp_warps_issue_stalled_')
              and not h[i].endswith('_not_issued')]
        tot = sum(float(b.replace(',', '') or 0) for _, b in st) or 1
        print('  stall samples (share):')
        for a, b in sorted(st, key=lambda t: -float(t[1].replace(',', '') or 0))[:8]:
            print(f'    {a[33:]:40s} {float(b.replace(",", "") or 0) / tot:6.1%}')


if __name__ == '__main__':
    main(sys.argv[1])
