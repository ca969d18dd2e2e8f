"""Top stall sites of one kernel from an ncu report's SASS source page.

  python tools/ncu_hot.py <report.ncu-rep> <kernel-regex> [top]
"""
import csv
import io
import subprocess
import sys


def main(rep, kern, top=25):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[start]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    body = [r for r in rows[start + 1:] if len(r) > si and r[si].isdigit()]
    total = sum(int(r[si]) for r in body) or 1
    for r in sorted(body, key=lambda r: -int(r[si]))[:int(top)]:
        print(f"{int(r[si]) * 100.0 / total:6.2f}%  {r[0]}  {r[1].strip()}")


if __name__ == "__main__":
    main(*sys.argv[1:])
