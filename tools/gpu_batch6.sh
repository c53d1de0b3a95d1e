#!/bin/bash
# GPU batch: parity subset + geometry test, headline bench, shard lines, source-level ncu at p=2048
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-v23}
timeout 900 python -m pytest tests/test_gpu_edge_cases.py tests/test_gpu_parity.py tests/test_gpu_probe.py -x -q > gpurun_out/t_$TAG.log 2>&1; echo rc=$? >> gpurun_out/t_$TAG.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-ttb > gpurun_out/b_$TAG.json 2> gpurun_out/b_$TAG.err
for p in 2048 4096 8192; do timeout 400 python bench.py --pop $p --steps 3 --warmup 3 --no-ttb --no-cpu-baseline > gpurun_out/shard_${TAG}_$p.json 2>&1; done
POP=2048 GENS=2 BUDGET=40000 timeout 900 ncu --set full --import-source on --clock-control none -k regex:^k_improve$ --launch-skip 1 -c 1 \
  -o gpurun_out/imp2k_$TAG -f python tools/probes/improve_probe.py > gpurun_out/imp2k_$TAG.log 2>&1
ncu -i gpurun_out/imp2k_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/imp2k_${TAG}_src.csv 2>&1
ncu -i gpurun_out/imp2k_$TAG.ncu-rep --page raw --csv > gpurun_out/imp2k_${TAG}_raw.csv 2>&1
[ -n "$TTB" ] && timeout 1500 python tools/ttb_hard.py --configs hard,c4 --pops $TTB --race-only --reference-from profiles/r02_ttb_hard.json > gpurun_out/ttb_$TAG.json 2> gpurun_out/ttb_$TAG.err
tail -2 gpurun_out/t_$TAG.log
