"""Host-side measurement tooling (CPU): the ncu kernel-name -> bench.py kernel-name mapping that
keys profiles/ncu_traffic.json (the bench line's roofline.traffic / issue_view), the launch-list
summary, and bench.py's algorithmic-bytes table covering every kernel the bench times."""
import csv
import io
import os
import sys
from contextlib import redirect_stdout

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import launch_summary  # noqa: E402
from ncu_summary import bench_name  # noqa: E402


def test_bench_name_mapping():
    cases = {
        "k_block_scatter<3, 0, 0, 0>": "p2g",
        "k_block_scatter<3, 1, 0, 0>": "g2p_T",
        "k_block_scatter<3, 0, 1, 0>": "p2g_fcr",
        "k_block_scatter<2, 1, 0, 1>": "g2p_T",
        "k_p2g_adj<3, 0, 0, 0>": "p2g_T",
        "k_p2g_adj<3, 1, 0, 0>": "p2g_T_massgrad",
        "k_p2g_adj<3, 0, 1, 0>": "p2g_T_fcr",
        "k_g2p<3, 0>": "g2p",
        "k_g2p2g<3, 0, 1, 1>": "g2p2g",
        "k_g2p2g<3, 0, 0, 1>": "g2p2g",
        "k_g2p2g<3, 0, 1, 0>": "g2p2g_last",
        "k_g2p2g<3, 1, 1, 1>": "g2p2g_fcr",
        "k_grid_adj<3>": "grid_T",
        "k_scan_lookback<3, 1>": "scan",
        "k_scatter": "scatter",
    }
    for k, v in cases.items():
        assert bench_name(k) == v, (k, bench_name(k), v)


def test_launch_summary_aggregates(tmp_path):
    rows = [["==PROF== noise"], ["ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"]]
    for i, (k, unit, val) in enumerate([("void mpm::k_p2g_adj<3, 0, 0, 0>(KParams, StepArgs)", "usecond", "150.0"),
                                        ("void mpm::k_p2g_adj<3, 0, 0, 0>(KParams, StepArgs)", "usecond", "154.0"),
                                        ("void mpm::k_g2p2g<3, 0, 1, 1>(KParams, StepArgs)", "nsecond", "132,000")]):
        rows.append([str(i), k, "gpu__time_duration.sum", unit, val])
    p = tmp_path / "launches.csv"
    with open(p, "w", newline="") as f:
        csv.writer(f, quoting=csv.QUOTE_ALL).writerows(rows)
    buf = io.StringIO()
    with redirect_stdout(buf):
        launch_summary.main(str(p))
    out = buf.getvalue().splitlines()
    assert "3 launches, 436.0 us total" in out[0]
    first = out[2].split()
    assert first[0] == "mpm::k_p2g_adj<3," and first[-3:] == ["304.0", "152.00", "0.697"]


def test_bench_alg_bytes_cover_timed_kernels():
    import bench
    for k in ("p2g", "g2p", "g2p2g", "p2g_T", "g2p_T", "grid_T"):
        bp, bn = bench.ALG_BYTES[k]
        assert bp >= 0 and bn > 0 and bp + bn > 0
    # the fused pass moves the unfused pair's particle bytes minus P2G's re-read of the state
    assert bench.ALG_BYTES["g2p2g"][0] == bench.ALG_BYTES["g2p"][0] + 20
