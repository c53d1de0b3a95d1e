#!/bin/bash
# full GPU test suite + headline bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-x}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t_$TAG.log 2>&1; echo rc=$? >> gpurun_out/t_$TAG.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/b_$TAG.json 2> gpurun_out/b_$TAG.err
tail -3 gpurun_out/t_$TAG.log
