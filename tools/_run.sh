timeout 900 python -m pytest tests/test_gpu_bucket.py tests/test_gpu_parity_extra.py tests/test_gpu_ops.py tests/test_gpu_backward_variants.py -x -q 2>&1 | tail -2
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-cache-bench > gpurun_out/sc.json 2>gpurun_out/sc.err; python tools/bline.py sc < gpurun_out/sc.json
