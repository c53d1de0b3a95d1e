#!/bin/bash
# GPU batch for the PLITS kernel: parity subset, steady-state probe (plain and PLSE_PROFILE), MPMA bench line
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-p1}
timeout 900 python -m pytest tests/test_gpu_plits.py tests/test_gpu_probe.py "tests/test_gpu_scale.py::test_c3_plits_slot_reuse" \
  tests/test_gpu_edge_cases.py -x -q > gpurun_out/pt_$TAG.log 2>&1; echo rc=$? >> gpurun_out/pt_$TAG.log
GENS=6 timeout 600 python tools/probes/plits_probe.py > gpurun_out/pp_$TAG.log 2>&1
PLSE_PROFILE=1 GENS=5 timeout 900 python tools/probes/plits_probe.py > gpurun_out/ppp_$TAG.log 2>&1
timeout 900 python bench.py --variant mpma --steps 5 --warmup 3 --no-ttb --no-cpu-baseline > gpurun_out/bm_$TAG.json 2> gpurun_out/bm_$TAG.err
tail -2 gpurun_out/pt_$TAG.log
if [ -n "$NCU" ]; then
  GENS=4 timeout 900 ncu --set full --import-source on --clock-control none -k regex:^k_plits --launch-skip 3 -c 1 \
    -o gpurun_out/plits4_$TAG -f python tools/probes/plits_probe.py > gpurun_out/plits4_$TAG.log 2>&1
  ncu -i gpurun_out/plits4_$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/plits4_${TAG}_src.csv 2>&1
  ncu -i gpurun_out/plits4_$TAG.ncu-rep --page raw --csv > gpurun_out/plits4_${TAG}_raw.csv 2>&1
fi
if [ -n "$TAIL" ]; then
  N=50 R=0.4 POP=8192 GENS=6 timeout 600 python tools/probes/improve_probe.py > gpurun_out/tail_c2_$TAG.log 2>&1
  POP=2048 GENS=6 timeout 600 python tools/probes/improve_probe.py > gpurun_out/tail_c3_2k_$TAG.log 2>&1
  N=50 R=0.4 POP=8192 GENS=4 PLSE_PROFILE=1 timeout 600 python tools/probes/improve_probe.py > gpurun_out/tail_c2p_$TAG.log 2>&1
fi
