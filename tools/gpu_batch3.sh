#!/bin/bash
# GPU batch: full gpu tests, shard-size bench lines, light ncu of k_improve at C3 16k, time-to-target
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t3.log 2>&1; echo rc=$? >> gpurun_out/t3.log
for p in 8192 4096 2048; do
  timeout 400 python bench.py --pop $p --steps 3 --warmup 3 --no-ttb --no-cpu-baseline > gpurun_out/shard_$p.json 2> gpurun_out/shard_$p.err
done
POP=16384 GENS=2 timeout 900 ncu --clock-control none -k regex:^k_improve$ --launch-skip 1 -c 1 \
  --section SpeedOfLight --section LaunchStats --section Occupancy --section WarpStateStats --section SchedulerStats \
  --metrics smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__inst_issued.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second \
  -o gpurun_out/imp16k_light -f python tools/probes/improve_probe.py > gpurun_out/imp16k_light.log 2>&1
ncu -i gpurun_out/imp16k_light.ncu-rep --page raw --csv > gpurun_out/imp16k_light_raw.csv 2>&1
timeout 3000 python tools/ttb_hard.py --configs hard,c4 --pops 16384 --limit 600 > gpurun_out/ttb_hard.json 2> gpurun_out/ttb_hard.err
tail -2 gpurun_out/t3.log
