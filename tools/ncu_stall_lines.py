"""Per-source-line warp-stall samples split by reason (top 3 per line) and executed
instructions, for one kernel of an ncu report (`--import-source on` capture):
  python tools/ncu_stall_lines.py report.ncu-rep <kernel-regex> [top]
Used for the round-2 analysis in DESIGN section 6 (which loads the P2G^T park removed, where
the G2P2G barrier waits sit)."""
import csv
import io
import subprocess
import sys

REASONS = ["stall_barrier", "stall_long_sb", "stall_short_sb", "stall_wait", "stall_math", "stall_mio",
           "stall_not_selected", "stall_selected", "stall_no_inst", "stall_dispatch", "stall_lg",
           "stall_branch_resolving", "stall_membar"]


def main(rep, kern, top=20):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                          "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = [i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r][0]
    h = rows[hi]
    idx = {r: h.index(r) for r in REASONS}
    ia, ie = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    lines, tot_r = [], {r: 0 for r in REASONS}
    for r in rows[hi + 1:]:
        if len(r) < len(h) or not r[0].strip().isdigit():
            continue
        try:
            tot, ni = int(r[ia] or 0), int(r[ie] or 0)
        except ValueError:
            continue
        d = {k: int(r[v] or 0) for k, v in idx.items()}
        for k in d:
            tot_r[k] += d[k]
        lines.append((tot, int(r[0]), r[1][:70], d, ni))
    lines.sort(reverse=True)
    T = sum(l[0] for l in lines) or 1
    TI = sum(l[4] for l in lines) or 1
    print({k[6:]: round(v / T, 3) for k, v in sorted(tot_r.items(), key=lambda x: -x[1]) if v / T > 0.005})
    for tot, ln, src, d, ni in lines[:top]:
        t3 = sorted(d.items(), key=lambda x: -x[1])[:3]
        print(ln, round(tot / T, 3), round(ni / TI, 3), src.strip()[:60], [(k[6:], v) for k, v in t3])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 20)
