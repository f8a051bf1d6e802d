"""Per-source-line stall samples and executed instructions for one kernel of an ncu report:
  python tools/ncu_lines.py report.ncu-rep <kernel-regex> [top] [skip] [--by-inst]"""
import csv
import io
import subprocess
import sys


def main(rep, kern, top=30, skip=0, by_inst=False):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                          "--launch-skip", str(skip), "--launch-count", "1", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = [i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r][0]
    h = rows[hi]
    ism, iex = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    lines = []
    for r in rows[hi + 1:]:
        if len(r) < len(h) or r[0] == "":
            continue
        try:
            lines.append((int(r[0]), r[1].strip()[:100], int(r[ism] or 0), int(r[iex] or 0)))
        except ValueError:
            continue
    tot_s = sum(l[2] for l in lines) or 1
    tot_i = sum(l[3] for l in lines) or 1
    print(f"samples {tot_s}  warp-instructions {tot_i}")
    key = (lambda l: -l[3]) if by_inst else (lambda l: -l[2])
    for ln, src, s, i in sorted(lines, key=key)[:top]:
        print(f"{ln:5d} stall {s / tot_s:6.3f} inst {i / tot_i:6.3f}  {src}")


if __name__ == "__main__":
    a = [x for x in sys.argv[1:] if not x.startswith("--")]
    main(a[0], a[1], int(a[2]) if len(a) > 2 else 30, int(a[3]) if len(a) > 3 else 0, "--by-inst" in sys.argv)
