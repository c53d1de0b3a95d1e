cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_refties.py tests/test_gpu_plits.py tests/test_gpu_edge_cases.py tests/test_gpu_probe.py -x -q > gpurun_out/t_v22.log 2>&1; echo rc=$? >> gpurun_out/t_v22.log
for p in 2048 4096 8192; do timeout 400 python bench.py --pop $p --steps 3 --warmup 3 --no-ttb --no-cpu-baseline > gpurun_out/shard_v22_$p.json 2>&1; done
timeout 400 python bench.py --variant mpma --steps 3 --warmup 3 --no-ttb --no-cpu-baseline > gpurun_out/mpma_v22.json 2>&1
tail -2 gpurun_out/t_v22.log
