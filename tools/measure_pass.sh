# measurement pass (run on the GPU box from the repo root; outputs under gpurun_out/): ncu full capture first
# (so the bench line's traffic and issue view use this build's counters), then bench lines, reference arm,
# small configs, paper cubes, ncu launch list
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
EXTRA=$(python tools/ncu_summary.py --metrics)
MPM_FUSE=1 python tools/time_step.py 10 > gpurun_out/ts_plain.json 2>&1 && \
MPM_FUSE=1 ncu --set full --metrics $EXTRA --import-source on --clock-control none \
    -k regex:'k_g2p2g|k_p2g_adj|k_block_scatter|k_grid_adj|k_scan_lookback|k_scatter' --launch-skip 24 -c 14 \
    -o gpurun_out/prof python tools/time_step.py 10 > gpurun_out/ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/prof.ncu-rep --traffic-json profiles/ncu_traffic.json --workload C4 > gpurun_out/ncu_summary.txt 2>&1
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python bench.py --workload C5a --no-cpu-baseline > gpurun_out/bench_c5a.json 2> gpurun_out/bench_c5a.err
python bench.py --workload C5b --no-cpu-baseline > gpurun_out/bench_c5b.json 2> gpurun_out/bench_c5b.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/reference.json 2> gpurun_out/reference.err
MPM_FUSE=1 python tools/small_configs.py > gpurun_out/small_configs.jsonl 2>&1
MPM_FUSE=1 python tools/paper_cubes.py > gpurun_out/paper_cubes.jsonl 2>&1
python bench.py --steps 15 --warmup 3 --no-cpu-baseline > gpurun_out/plain_launches.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 15 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
echo done
