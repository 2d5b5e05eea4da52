"""Warp-stall samples per CUDA source line from an ncu report (dev tool):
SASS rows of the mixed cuda,sass source page attributed to the CUDA line
they follow.  python tools/ncu_lines.py x.ncu-rep [top]"""
import csv
import subprocess
import sys
from collections import defaultdict


def main(path, top=40):
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                         capture_output=True, text=True).stdout
    f, line, src, hdr = None, None, '', None
    agg = defaultdict(float)
    srcs = {}
    total = 0.0
    for r in csv.reader(out.splitlines()):
        if len(r) == 2 and r[0] == 'File Path':
            f = r[1].split('/')[-1]
            continue
        if r and r[0] == 'Line No':
            hdr = r
            continue
        if not hdr or len(r) < 5:
            continue
        if r[0].isdigit():
            line, src = int(r[0]), r[1].strip()
        col = 4   # "Warp Stall Sampling (All Samples)"
        try:
            s = float(r[col])
        except ValueError:
            continue
        if r[0] == '' and line is not None:
            agg[(f, line)] += s
            srcs[(f, line)] = src
            total += s
    for (f, ln), s in sorted(agg.items(), key=lambda a: -a[1])[:top]:
        print(f"{s / total * 100:5.1f}%  {f}:{ln:<5d} {srcs[(f, ln)][:100]}")


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
