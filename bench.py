#!/usr/bin/env python
"""Benchmark of the differentiable MLS-MPM step (ChainQueen, arXiv 1810.01054) on B200.

Metric (BASELINE.json): particle-steps/s, forward + backward, 3D, at N GPUs; HBM GB/s as a
fraction of the measured peak for the dominant kernel.

Workload (N = 1 and per rank for N > 1): configs[3] "C4" -- 3D 128^3 grid, 1,048,576-particle
neo-Hookean slab (64x32x64 cells, 8 particles per cell, v0 = (0,-1,0), 8 octant actuators,
dt = 1e-4).  One "step" = one forward MLS-MPM step (binning, P2G, grid update, G2P) plus its
reverse-mode step (G2P^T, grid^T, P2G^T) -- every row of SURVEY 8(a).  K steps = forward K
steps onto the tape, then the backward pass over those K steps (loss: final CoM x).
Multi-GPU: each rank runs its own independent C4 rollout (weak scaling, no data-path
collective); the barrier / max-over-ranks timing uses torch.distributed.
--workload C5b: 64 quadruped rollouts sharded over ranks (strong scaling, no collective).
--workload C5a: ONE 8,355,840-particle slab at 256^3 sharded by x-slab (strong scaling; the
grid windows at slab boundaries are summed with NCCL send/recv inside libmpm every step).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload C4|C5a|C5b]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1810_01054_b200 import parallel, scenes  # noqa: E402

METRIC = "particle-steps/sec fwd and fwd+bwd (3D, 1/2/4/8 B200); HBM GB/s % peak"
UNIT = "particle-steps/s"
WORKLOADS = {
    "C4": ("C4 (configs[3]): 3D 128^3 grid, 1,048,576-particle neo-Hookean slab, "
           "forward+backward, loss = final CoM x; one rollout per rank"),
    "C5b": ("C5b (configs[4] batch part): 64 independent 3D 64^3 quadruped rollouts "
            "(29,952 particles each, per-rollout actuation phase and E scale), sharded over ranks"),
    "C5a": ("C5a (configs[4] slab part): one 3D 256^3 slab of 240x32x136 cells, 8,355,840 particles, "
            "dt = 5e-5, forward+backward, loss = final CoM x; x-slab sharded over ranks with halo "
            "window exchange"),
}
SEG = 200  # max steps per tape segment (tape memory ~ 100 MB per step at C4)


def _cfg_dict(K, W, n_gpus, sc, workload="C4", slabs=None, fuse=0):
    par = "single GPU"
    if n_gpus > 1:
        par = (f"x-slab sharded x{n_gpus}, slabs {slabs}, NCCL halo-window sums" if workload == "C5a"
               else f"rollout-sharded x{n_gpus} (no data-path collective)")
    return {"workload": WORKLOADS[workload], "particles_per_rank": int(sc.batch * sc.n),
            "rollouts_per_rank": int(sc.batch), "grid": f"{sc.res}^3", "dim": 3, "dt": sc.dt,
            "steps_per_pass": K, "warmup": W, "parallelism": par,
            "forward": ("fused G2P2G, one particle pass per step (NEXT N2)"
                        + ("; slab windows of grid t+1 summed between launches" if workload == "C5a" and n_gpus > 1 else "")
                        if fuse else "P2G + G2P passes"),
            "l2": (f"inputs larger than L2: per-step state {sc.batch * sc.n * 96 / 2**20:.0f} MiB read + written, "
                   f"tape of K states")}


def make_scene(workload, rank, world, tape):
    """(this rank's scene, total particles of the job, slab bounds or None, total mass per
    rollout for the CoM seed or None)."""
    if workload == "C4":
        sc = scenes.slab_3d(seed=rank, steps=tape)
        return sc, sc.n * world, None, None
    if workload == "C5a":
        full = scenes.slab_c5a(seed=0, steps=tape)
        bounds = parallel.slab_partition(full.x[0], full.res, full.dim, world)
        sc, _ = parallel.shard_slab(full, *bounds[rank])
        return sc, full.n, bounds, float(full.mass.astype(np.float64).sum())
    full = scenes.quadruped_3d(seed=0, batch=64, steps=tape, e_scale=True)
    return parallel.shard_scene(full, parallel.Dist(rank, world)), 64 * full.n, None, None


# ---------------------------------------------------------------------------------------
# clocks during the timed region (NVML, sampled in a thread)
# ---------------------------------------------------------------------------------------
class ClockSampler:
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle",
               0x2: "applications_clocks_setting", 0x10: "sync_boost"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def _peaks():
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


# Algorithmic bytes per launch: what each kernel must move, per
# particle (NT) and per touched grid node (TN), fp32.
ALG_BYTES = {
    "p2g": (96 + 20, 16),          # read x,v,C,F + m,V,mu,lam,aid ; write (p,m) per node
    "g2p": (48 + 96, 16),          # read x,F + write x,v,C,F ; read (vbar,m) per node
    "p2g_T": (96 + 20 + 96 + 96 + 16, 32),  # tape state, params, adj in, adj out, dmu/dlam RMW ; tape + adj node
    "g2p_T": (48 + 96, 16),        # x,F + adj in ; write dv per node
    "grid_T": (0, 48),
    "g2p2g": (48 + 96 + 20, 32),   # fused (NEXT N2): read x,F + write x,v,C,F + params ; read grid t, write grid t+1
}


def _ncu(field, kernel, workload):
    """`field` per launch of `kernel` from the committed ncu capture (profiles/
    ncu_traffic.json) when it was taken on this workload, else None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(path))
        return d[field][kernel] if d.get("workload") == workload else None
    except Exception:
        return None


def _traffic(kernel, workload):
    return _ncu("per_launch_dram_bytes", kernel, workload)


# The paper's own speed numbers (Table I): context, not a target --
# another GPU (GTX 1080 Ti), a falling cube whose grid, dt, E, nu are not printed, "time
# per frame" read as one step per frame.  vs_baseline stays null (BASELINE.json publishes none).
PAPER_TABLE_I = {
    "hardware": "NVIDIA GTX 1080 Ti (PAPER.md:183)", "source": "PAPER.md:190-197, Table I (3D falling cube)",
    "assumption": "1 MLS-MPM step per frame (the paper does not say)",
    "cubes": {str(n): {"fwd_ms": f, "bwd_ms": b, "fwd_bwd_particle_steps_per_s": round(n / ((f + b) * 1e-3))}
              for n, f, b in ((8000, 0.392, 0.406), (64000, 1.594, 1.774), (512000, 10.501, 11.594))},
}


# ---------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------
def run_ours(args):
    import torch

    from paper_1810_01054_b200 import mpm

    # MPM_BENCH_SHARED_GPU=1 (tests only): the ranks share cuda:0 and talk through gloo (slab
    # exchanges through a host-staged transport) -- checks the N > 1 harness on a 1-GPU box;
    # its timings mean nothing
    shared = os.environ.get("MPM_BENCH_SHARED_GPU") == "1"
    D = parallel.init_from_env("gloo" if shared else ("nccl" if int(os.environ.get("WORLD_SIZE", "1")) > 1 else None))
    world, rank, local = D.world, D.rank, D.local_rank
    dev = torch.device("cuda", local if world > 1 and not shared else 0)
    torch.cuda.set_device(dev)
    K, W = args.steps, args.warmup
    seg = min(K, SEG)
    tape = max(seg, min(W, SEG), 1)
    sc, total_particles, slabs, mtot = make_scene(args.workload, rank, world, tape)
    stream = torch.cuda.current_stream(dev)
    sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=tape, device=dev.index, stream=stream.cuda_stream,
                                        fuse_g2p2g=args.fuse))
    if slabs is not None:
        sim.set_slab(*slabs[rank], 1)
        if world > 1:
            if shared:
                sim.set_transport(parallel.gloo_transport(D))
            else:
                parallel.init_slab_comm(sim, D)
    NT = sc.batch * sc.n
    m = torch.tensor(sc.mass, device=dev, dtype=torch.float64)  # [B][N]
    seed = torch.zeros((NT, 3), device=dev, dtype=torch.float32)
    msum = m.sum(dim=1, keepdim=True) if mtot is None else mtot  # whole-body mass in slab mode
    seed[:, 0] = (m / msum).reshape(-1).float()  # CoM_x of each rollout
    sim.set_scene(sc)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)

    def passes(n_steps, fwd_events=None):
        left = n_steps
        while left > 0:
            s = min(left, seg)
            sim.rewind(0)
            sim.forward(s)
            if fwd_events is not None:
                fwd_events.append(torch.cuda.Event(enable_timing=True))
                fwd_events[-1].record(stream)
            sim.backward(seed)
            left -= s

    # warm-up: W steps (forward + backward), untimed
    passes(max(W, 1))
    # timed region: exactly K steps
    barrier()
    n0 = sim.launches
    with ClockSampler(dev.index) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        fwd_ev = []
        e0.record(stream)
        passes(K, fwd_ev)
        e1.record(stream)
        barrier()
    launches = sim.launches - n0
    ms = e0.elapsed_time(e1)
    fwd_ms = e0.elapsed_time(fwd_ev[0]) if len(fwd_ev) == 1 else None
    ms = parallel.max_over_ranks(ms, D, dev)
    fwd_ms = parallel.max_over_ranks(fwd_ms, D, dev) if fwd_ms is not None else None
    value = total_particles * K / (ms / 1e3)

    # roofline: per-kernel CUDA-event times of a second, profiled pass of the same K steps
    sim.set_profiling(True)
    passes(K)
    prof = sim.profile()
    sim.set_profiling(False)
    steps_info = [sim.step_info(t_)[1] for t_ in range(sim.tape_length)]
    TN = float(np.mean(steps_info)) * 64
    peak, peak_src = _peaks()
    per_kernel = {}
    for kname, (ms_k, n_k) in prof.items():
        if n_k == 0:
            continue
        ent = {"ms_total": round(ms_k, 4), "launches": n_k, "us_per_launch": round(1e3 * ms_k / n_k, 2)}
        if kname in ALG_BYTES:
            bp, bn = ALG_BYTES[kname]
            byt = bp * NT + bn * TN
            ent["alg_bytes_per_launch"] = int(byt)
            ent["gbs"] = round(byt / (ms_k / n_k * 1e-3) / 1e9, 1)
        per_kernel[kname] = ent
    dom = max((k for k in per_kernel if k in ALG_BYTES), key=lambda k: per_kernel[k]["ms_total"])
    d = per_kernel[dom]
    prof_total = sum(v["ms_total"] for v in per_kernel.values())
    roofline = {"bound": "hbm", "kernel": dom, "achieved": d["gbs"], "peak": peak, "unit": "GB/s",
                "frac": round(d["gbs"] / peak, 4), "traffic": _traffic(dom, args.workload),
                "peak_source": peak_src, "share_of_step": round(d["ms_total"] / prof_total, 3),
                "alg_bytes_per_launch": d["alg_bytes_per_launch"],
                "per_kernel": per_kernel}
    # issue view (these kernels are latency / issue bound): warp instructions per launch from
    # the committed ncu capture over 4 schedulers x SMs x the max SM clock, vs the measured time
    inst = _ncu("per_launch_warp_instructions", dom, args.workload)
    if inst:
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        floor_us = inst / (4 * sms * 1965e6) * 1e6
        roofline["issue_view"] = {"warp_instructions_per_launch": inst, "issue_floor_us": round(floor_us, 1),
                                  "measured_us": d["us_per_launch"], "frac": round(floor_us / d["us_per_launch"], 3)}

    # e2e through the public API with pinned host buffers: set_state (H2D), forward,
    # backward (seed H2D), grad (D2H), every pass
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    h_in = [pin(a.reshape(NT, *a.shape[2:])) for a in (sc.x, sc.v, sc.F, sc.C, sc.mass, sc.vol, sc.E, sc.nu, sc.actuator_id)]
    act = np.zeros((sc.batch, tape, sc.n_act, 3), np.float32)
    act[:, :min(tape, sc.act.shape[1])] = sc.act[:, :tape]
    h_act = pin(act)
    h_seed = pin(seed.cpu().numpy())
    h_out = {k: torch.empty(s, dtype=torch.float32).pin_memory() for k, s in
             (("dx0", (NT, 3)), ("dv0", (NT, 3)), ("dF0", (NT, 3, 3)), ("dC0", (NT, 3, 3)),
              ("dE", (NT,)), ("dnu", (NT,)), ("da", (sc.batch, tape, sc.n_act, 3)))}
    h2d = sum(a.numel() * a.element_size() for a in h_in) + h_act.numel() * 4
    d2h = sum(a.numel() * a.element_size() for a in h_out.values())
    barrier()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    left = K
    nseg = 0
    while left > 0:
        s = min(left, seg)
        sim.set_state(*h_in)
        sim.set_actuation(h_act)
        sim.forward(s)
        sim.backward(h_seed)
        sim.grad(h_out)
        left -= s
        nseg += 1
    e3.record(stream)
    barrier()
    e2e_ms = e2.elapsed_time(e3)
    e2e_ms = parallel.max_over_ranks(e2e_ms, D, dev)
    e2e = {"value": total_particles * K / (e2e_ms / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": int((h2d + h_seed.numel() * 4) * nseg / K),
           "d2h_bytes_per_step": int(d2h * nseg / K)}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": ms / K, "higher_is_better": True,
            "scaling": "weak" if args.workload == "C4" else "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded jittered-lattice slab)",
            "config": _cfg_dict(K, W, world, sc, args.workload, slabs, args.fuse),
            "fwd": {"value": (total_particles * K / (fwd_ms / 1e3)) if fwd_ms else None,
                    "ms_per_step": (fwd_ms / K) if fwd_ms else None},
            "roofline": roofline, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(), "paper": PAPER_TABLE_I}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if args.workload == "C4":
            line["cpu_baseline"] = cpu_baseline_full(sc)
        elif args.workload == "C5a":  # bounded sample: a 1M-particle sub-slab at the same res/density
            line["cpu_baseline"] = cpu_baseline_full(
                scenes.slab_3d(steps=1, cells=(64, 32, 64), res=256, y0=10, dt=5e-5), "C5a sub-slab 64x32x64 cells")
        else:
            line["cpu_baseline"] = cpu_baseline_full(scenes.quadruped_3d(steps=1), "one C3 quadruped rollout")
    sim.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


# ---------------------------------------------------------------------------------------
# oracle legs (CPU): cpu_baseline of our line, and the --impl reference arm
# ---------------------------------------------------------------------------------------
def cpu_info():
    """CPU model (/proc/cpuinfo, as lscpu reports it), logical CPUs and the CPUs this process may use."""
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count()
    return {"cpu_model": model, "logical_cpus": os.cpu_count(), "usable_cpus": usable}


def _oracle_fb(sc, n_steps, variant="serial64"):
    """Forward n_steps + backward (seed: CoM_x) of rollout 0 with one oracle build: serial64 (the
    oracle as it stands), serial32, omp64, omp32 (oracle.forward_backward_timing)."""
    import oracle
    cfg = oracle.Config(dim=sc.dim, res=sc.res, dt=sc.dt, gravity=sc.gravity, bound=sc.bound,
                        friction=sc.friction, act_strength=sc.act_strength, n_act=sc.n_act)
    st = oracle.pack(sc.x[0], sc.v[0], sc.C[0], sc.F[0])
    prm = [a[0].astype(np.float64) for a in (sc.mass, sc.vol, sc.E, sc.nu)]
    act = sc.act[0][:max(n_steps, 1)].astype(np.float64)
    seed = np.zeros_like(st)
    seed[:, 0] = prm[0] / prm[0].sum()
    f, fb, _ = oracle.forward_backward_timing(cfg, st, *prm, sc.actuator_id[0], act, seed, n_steps, variant)
    return f, fb


def cpu_baseline_full(sc, what="full C4 state"):
    """The CPU oracle timed on this host: 1 forward + 1 backward step of the given
    state with the serial fp64 oracle as it stands, its fp32 build, and the OpenMP builds (fp64
    and fp32) at all usable cores with fixed-order merges of per-chunk grids.  value = the OpenMP
    fp64 rate (the fair multithreaded CPU number); ~15-40 s of CPU work in total."""
    import oracle
    n = sc.batch * sc.n
    rates = {}
    for v in ("omp64", "omp32", "serial64", "serial32"):
        f, fb = _oracle_fb(sc, 1, v)
        rates[v] = {"fwd_bwd": n / fb, "fwd": n / f}
    threads = oracle.omp_threads()
    info = cpu_info()
    return {"value": rates["omp64"]["fwd_bwd"], "unit": UNIT, "cores": threads, "threads": threads,
            "kind": "oracle", **info,
            "fp64": {"threads": rates["omp64"], "1_thread": rates["serial64"]},
            "fp32": {"threads": rates["omp32"], "1_thread": rates["serial32"]},
            "sample": f"{what} ({n} particles), 1 forward + 1 backward step per variant; value = fp64 OpenMP "
                      f"build at {threads} threads (per-chunk scatter grids merged in fixed order); the serial fp64 "
                      f"oracle as it stands: {rates['serial64']['fwd_bwd']:.4g} particle-steps/s"}


REF_BUDGET_S = 150.0  # wall-clock budget of the reference arm's timed steps


def run_reference(args):
    """--impl reference: the CPU oracle (fp64, OpenMP build at all usable cores) on the same
    metric / config / unit.  Each step is one forward + one backward step of the FULL C4 state
    (1,048,576 particles, the bench workload) when K steps fit REF_BUDGET_S; otherwise of a
    sub-slab of the same slab at the same density, sized to fit."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        # torchrun sets OMP_NUM_THREADS=1 per rank; rank 0 runs the oracle alone here, on all
        # the cores it may use (set before the OpenMP runtime is loaded)
        os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
    import oracle
    K, W = args.steps, args.warmup
    full = scenes.slab_3d(seed=0, steps=2)
    f, fb = _oracle_fb(full, 1, "omp64")  # first warm-up step, on the full state
    sc, cells = full, (64, 32, 64)
    if fb * K > REF_BUDGET_S:
        for cells in ((32, 32, 64), (32, 16, 32), (16, 16, 16), (8, 8, 8)):
            if fb * K * (cells[0] * cells[1] * cells[2]) / (64 * 32 * 64) <= REF_BUDGET_S:
                break
        sc = scenes.slab_3d(seed=0, steps=2, cells=cells)
    n = sc.batch * sc.n
    for _ in range(W - 1):
        _oracle_fb(sc, 1, "omp64")
    t0 = time.perf_counter()
    for _ in range(K):
        _oracle_fb(sc, 1, "omp64")
    dt = time.perf_counter() - t0
    value = n * K / dt
    threads = oracle.omp_threads()
    what = ("the full C4 state" if sc is full else
            f"a sub-slab {cells[0]}x{cells[1]}x{cells[2]} cells of the C4 slab at the same density")
    sample = (f"{what} ({n} particles, 128^3 grid), 1 forward + 1 backward step per step, fp64, OpenMP build "
              f"at {threads} threads")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": K, "warmup": W, "ms_per_step": 1e3 * dt / K, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded jittered-lattice slab)",
            "config": {**_cfg_dict(K, W, args.gpus, full, "C4"), "same_config": sc is full},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "threads": threads, "kind": "oracle",
                             "sample": sample, **cpu_info()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)  # ~80 ms timed at C4: enough in-region clock samples
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="C4", choices=sorted(WORKLOADS))
    ap.add_argument("--fuse", type=int, default=1, choices=[0, 1],
                    help="fused G2P2G forward (NEXT N2; C5a split over GPUs sums grid t+1's windows between launches)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
