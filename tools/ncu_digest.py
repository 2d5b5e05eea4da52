"""Digest of an ncu --set full capture (dev tool): the metrics the profiles/
summaries quote, plus the top stall reasons.  python tools/ncu_digest.py x.ncu-rep"""
import csv
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'launch__grid_size', 'launch__block_size', 'launch__registers_per_thread',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sector_hit_rate.pct',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'dram__throughput.avg.pct_of_peak_sustained_elapsed']


def main(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    for v in vals:
        print('kernel:', v[hdr.index('Kernel Name')])
        for w in WANT:
            if w in hdr:
                print(f"  {w:66s} {v[hdr.index(w)]:>16s} {units[hdr.index(w)]}")
        st = [(h, float(x or 0)) for h, x in zip(hdr, v)
              if h.startswith('smsp__pcsamp_warps_issue_stalled') and not h.endswith('not_issued')]
        tot = sum(x for _, x in st) or 1.0
        for h, x in sorted(st, key=lambda a: -a[1])[:10]:
            print(f"  {h:66s} {x:16.0f} ({x / tot * 100:.1f}%)")


if __name__ == '__main__':
    main(sys.argv[1])
