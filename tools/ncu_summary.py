"""Key counters per captured kernel from an ncu report (--page raw --csv):
  python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--traffic-json profiles/ncu_traffic.json --workload C4]
      [--allow-missing]
--traffic-json writes dram__bytes_read.sum + dram__bytes_write.sum per launch (mean over the
captured launches of each kernel), keyed by bench.py's kernel names (roofline "traffic").

Every counter in KEYS must be in the report: `--set full` does not collect the L2 reduction /
atomic counters, so the capture command adds them explicitly (EXTRA_METRICS, printed by
`python tools/ncu_summary.py --metrics`).  A missing counter is an error (exit 2) unless
--allow-missing is given -- a summary must not silently drop the evidence it is meant to carry."""
import csv
import io
import json
import subprocess
import sys

def bench_name(kernel):
    """bench.py's name of a captured kernel, from its template arguments (robust to added
    defaulted parameters such as the small-problem SPLIT flag)."""
    import re
    m = re.match(r"(\w+)(?:<([^>]*)>)?", kernel)
    base, args = m.group(1), [a.strip() for a in (m.group(2) or "").split(",") if a.strip()]
    flag = lambda i: len(args) > i and args[i] in ("1", "true")
    if base == "k_block_scatter":
        return ("g2p_T" if flag(1) else "p2g") + ("_fcr" if flag(2) else "")
    if base == "k_p2g_adj":
        return "p2g_T" + ("_massgrad" if flag(1) else "") + ("_fcr" if flag(2) else "")
    if base == "k_g2p2g":
        return "g2p2g" + ("_fcr" if len(args) > 1 and args[1] == "1" else "") + ("" if flag(3) else "_last")
    return {"k_g2p": "g2p", "k_grid_adj": "grid_T", "k_scan_lookback": "scan", "k_scatter": "scatter"}.get(base, kernel)


KEYS = [
    ("time_us", "gpu__time_duration.sum", "us"),
    ("dram_rd_MB", "dram__bytes_read.sum", "MB"),
    ("dram_wr_MB", "dram__bytes_write.sum", "MB"),
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
    ("red_req_K", "lts__t_requests_op_red.sum", 1e-3),
    ("l1_red_req_K", "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum", 1e-3),
    ("l1_atom_req_K", "l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum", 1e-3),
    ("shared_wf_M", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1e-6),
]
# counters outside `--set full` that the capture must request with --metrics (sm_100 names,
# checked with `ncu --query-metrics --chip gb100`)
EXTRA_METRICS = ["lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum", "lts__t_requests_op_red.sum",
                 "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum",
                 "l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum"]


TO_US = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}
TO_MB = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "KB": 1e-3, "MB": 1.0, "GB": 1e3}


def _scale(sc, unit):
    if sc == "us":
        return TO_US.get(unit, 1.0)
    if sc == "MB":
        return TO_MB.get(unit, 1.0)
    return sc


def main(rep, traffic_json=None, allow_missing=False):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    missing = [key for _, key, _ in KEYS if key not in hdr]
    if missing and not allow_missing:
        sys.stderr.write("ncu_summary: counters missing from the report (capture with --set full --metrics "
                         + ",".join(EXTRA_METRICS) + "): " + ", ".join(missing) + "\n")
        sys.exit(2)
    traffic = {}
    instr = {}
    stall = [i for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_")
             and h.endswith("_per_issue_active.ratio")]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
        out = []
        for short, key, sc in KEYS:
            if key in hdr and r[hdr.index(key)] not in ("", "n/a"):
                i = hdr.index(key)
                out.append(f"{short}={float(r[i].replace(',', '')) * _scale(sc, units[i]):.4g}")
            elif not allow_missing:
                sys.stderr.write(f"ncu_summary: {key} has no value for {name}\n")
                sys.exit(2)
        try:
            b = sum(float(r[hdr.index(k)].replace(",", "")) * TO_MB.get(units[hdr.index(k)], 1.0) * 1e6
                    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            traffic.setdefault(bench_name(name), []).append(b)
            inst = float(r[hdr.index("smsp__inst_executed.sum")].replace(",", ""))
            instr.setdefault(bench_name(name), []).append(inst)
        except (ValueError, IndexError):
            pass
        st = sorted(((hdr[i][34:-27], float(r[i] or 0)) for i in stall), key=lambda x: -x[1])[:5]
        print(name)
        print("   " + " ".join(out))
        print("   stalls: " + " ".join(f"{k}={v:.2f}" for k, v in st))
    if traffic_json:
        per = {k: round(sum(v) / len(v)) for k, v in traffic.items()}
        json.dump({"source": rep, "workload": WORKLOAD, "per_launch_dram_bytes": per,
                   "per_launch_warp_instructions": {k: round(sum(v) / len(v)) for k, v in instr.items()},
                   "captured_launches": {k: len(v) for k, v in traffic.items()}}, open(traffic_json, "w"), indent=1)


WORKLOAD = "C4"

if __name__ == "__main__":
    if "--metrics" in sys.argv:
        print(",".join(EXTRA_METRICS))
        sys.exit(0)
    tj = sys.argv[sys.argv.index("--traffic-json") + 1] if "--traffic-json" in sys.argv else None
    if "--workload" in sys.argv:
        WORKLOAD = sys.argv[sys.argv.index("--workload") + 1]
    main(sys.argv[1], tj, "--allow-missing" in sys.argv)
