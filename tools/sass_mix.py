"""Executed-instruction mix by SASS opcode for one kernel of an ncu report (source page, sass):
  python tools/sass_mix.py report.ncu-rep <kernel-regex> [top]"""
import collections
import csv
import io
import subprocess
import sys


def main(rep, kern, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                          "--launch-count", "1", "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    isrc, iex, ith = h.index("Source"), h.index("Instructions Executed"), h.index("Thread Instructions Executed")
    mix = collections.Counter()
    tmix = collections.Counter()
    for r in rows[2:]:
        if len(r) <= iex:
            continue
        op = r[isrc].strip().split()
        if not op:
            continue
        o = op[0] if not op[0].startswith("@") else op[1]
        o = o.split(".")[0]
        if not (r[iex] or "0").isdigit():
            continue
        mix[o] += int(r[iex] or 0)
        tmix[o] += int(r[ith] or 0)
    tot = sum(mix.values())
    print(f"warp instructions {tot}")
    for o, n in mix.most_common(top):
        print(f"{o:10s} {n / tot:6.3f}  active-lanes {tmix[o] / max(n, 1):5.1f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
