#!/bin/bash
# Round-2 evidence batch for the final kernel build: GPU tests, headline bench, BASELINE config lines,
# MPMA line, ncu light capture of k_improve at C3 16k -> summary keyed by source hash, launch list,
# K3 capture.  Everything lands in gpurun_out/ (merged back by gpurun).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-final}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t_$TAG.log 2>&1; echo rc=$? >> gpurun_out/t_$TAG.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/b_$TAG.json 2> gpurun_out/b_$TAG.err
timeout 600 python bench.py --n 50 --r 0.4 --pop 8192 --steps 5 --warmup 3 --no-ttb --no-cpu-baseline > gpurun_out/c2_$TAG.json 2>&1
timeout 600 python bench.py --n 70 --r 0.6 --pop 4096 --steps 3 --warmup 3 --no-ttb --no-cpu-baseline > gpurun_out/c4shard_$TAG.json 2>&1
timeout 900 python bench.py --lsc --n 70 --r 0.4 --seed 7 --pop 16384 --steps 3 --warmup 3 --no-ttb --no-cpu-baseline > gpurun_out/c5_$TAG.json 2>&1
timeout 900 python bench.py --variant mpma --steps 3 --warmup 3 --no-ttb --no-cpu-baseline > gpurun_out/mpma_$TAG.json 2>&1
POP=16384 GENS=2 timeout 900 ncu --clock-control none -k regex:^k_improve$ --launch-skip 1 -c 1 \
  --section SpeedOfLight --section LaunchStats --section Occupancy --section WarpStateStats --section SchedulerStats \
  --metrics smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__inst_issued.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second \
  -o gpurun_out/imp16k_$TAG -f python tools/probes/improve_probe.py > gpurun_out/imp16k_$TAG.log 2>&1
ncu -i gpurun_out/imp16k_$TAG.ncu-rep --page raw --csv > gpurun_out/imp16k_${TAG}_raw.csv 2>&1
GEN=2 python tools/probes/ncu_summary.py gpurun_out/imp16k_${TAG}_raw.csv gpurun_out/imp16k_$TAG.log k_improve \
  n60_r0.5_s12345_p16384_b180000 gpurun_out/k_improve_ncu_summary.json > gpurun_out/ncu_summary_$TAG.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 1 --no-ttb --no-cpu-baseline > gpurun_out/launches_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_sim_tc --launch-skip 2 -c 1 -o gpurun_out/k3_$TAG -f \
  python bench.py --steps 1 --warmup 1 --no-ttb --no-cpu-baseline > gpurun_out/k3_$TAG.log 2>&1
ncu -i gpurun_out/k3_$TAG.ncu-rep --page raw --csv > gpurun_out/k3_${TAG}_raw.csv 2>&1
PLSE_BENCH_DIST=gloo PLSE_BENCH_ONE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --pop 4096 --steps 2 --warmup 3 --no-ttb \
  --no-cpu-baseline > gpurun_out/functional_2rank_$TAG.json 2> gpurun_out/functional_2rank_$TAG.err
tail -2 gpurun_out/t_$TAG.log
