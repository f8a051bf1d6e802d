"""Key counters per captured kernel from an ncu report (--page raw --csv):
  python tools/ncu_summary.py gpurun_out/prof.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("time_us", "gpu__time_duration.sum", 1e-3),
    ("dram_rd_MB", "dram__bytes_read.sum", 1e-6),
    ("dram_wr_MB", "dram__bytes_write.sum", 1e-6),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("sm_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("l1_pct", "l1tex__throughput.avg.pct_of_peak_sustained_active", 1),
    ("l2_pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("warps_pct", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("regs", "launch__registers_per_thread", 1),
    ("inst_M", "smsp__inst_executed.sum", 1e-6),
    ("ipc", "sm__inst_executed.avg.per_cycle_active", 1),
    ("l1_hit", "l1tex__t_sector_hit_rate.pct", 1),
    ("l2_hit", "lts__t_sector_hit_rate.pct", 1),
    ("red_sect_K", "lts__t_sectors_op_red.sum", 1e-3),
    ("atom_sect_K", "lts__t_sectors_op_atom.sum", 1e-3),
    ("shared_wf_M", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1e-6),
]


def main(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    stall = [i for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_")
             and h.endswith("_per_issue_active.ratio")]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
        out = []
        for short, key, sc in KEYS:
            if key in hdr and r[hdr.index(key)] not in ("", "n/a"):
                out.append(f"{short}={float(r[hdr.index(key)].replace(',', '')) * sc:.4g}")
        st = sorted(((hdr[i][34:-27], float(r[i] or 0)) for i in stall), key=lambda x: -x[1])[:5]
        print(name)
        print("   " + " ".join(out))
        print("   stalls: " + " ".join(f"{k}={v:.2f}" for k, v in st))


if __name__ == "__main__":
    main(sys.argv[1])
