#!/bin/bash
# GPU batch: full gpu tests, headline bench, shard bench, light ncu of k_improve at C3 16k (instructions/move)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-v21}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_$TAG.log 2>&1; echo rc=$? >> gpurun_out/t_$TAG.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-ttb > gpurun_out/b_$TAG.json 2> gpurun_out/b_$TAG.err
timeout 400 python bench.py --pop 2048 --steps 3 --warmup 3 --no-ttb --no-cpu-baseline > gpurun_out/b2048_$TAG.json 2>&1
POP=16384 GENS=2 timeout 900 ncu --clock-control none -k regex:^k_improve$ --launch-skip 1 -c 1 \
  --section SpeedOfLight --section LaunchStats --section Occupancy --section WarpStateStats --section SchedulerStats \
  --metrics smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__inst_issued.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second \
  -o gpurun_out/imp16k_$TAG -f python tools/probes/improve_probe.py > gpurun_out/imp16k_$TAG.log 2>&1
ncu -i gpurun_out/imp16k_$TAG.ncu-rep --page raw --csv > gpurun_out/imp16k_${TAG}_raw.csv 2>&1
tail -2 gpurun_out/t_$TAG.log
