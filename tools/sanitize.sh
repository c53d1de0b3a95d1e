#!/bin/bash
# compute-sanitizer racecheck + synccheck (+ memcheck) of the four improve kernels and the population
# phases on small populations.  Logs -> gpurun_out/sanitizer_*.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in racecheck synccheck memcheck; do
  for v in "partial 0 0" "partial 0 32" "partial 1 0" "mpma 0 0" "mpma 1 0"; do
    set -- $v
    tag=${tool}_${1}_tie$2_wpc$3
    PLSE_IMPROVE_WPC=$3 N=20 R=0.5 POP=64 GENS=2 BUDGET=1500 VARIANT=$1 TIE=$2 timeout 900 $CS --tool $tool --print-limit 20 \
      python tools/probes/improve_probe.py > gpurun_out/sanitizer_$tag.log 2>&1
    echo "$tag rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitizer_$tag.log | tr '\n' ' ')"
  done
done
