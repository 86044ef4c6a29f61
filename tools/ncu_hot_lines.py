"""Hottest CUDA source lines (warp-stall samples) of one kernel in an ncu report.

    python tools/ncu_hot_lines.py report.ncu-rep kernel_regex [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 12
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                          "--launch-count", "1", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    src = [x for x in rows if len(x) > 5 and x[0].isdigit() and x[4].isdigit()]
    tot = sum(int(x[4]) for x in src) or 1
    src.sort(key=lambda x: -int(x[4]))
    for x in src[:top]:
        print(f"{x[0]:>5} {int(x[4]):>7} {100 * int(x[4]) / tot:5.1f}%  {x[1].strip()[:110]}")


if __name__ == "__main__":
    main()
