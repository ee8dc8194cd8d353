timeout 900 python -m pytest tests/test_gpu_bucket.py tests/test_gpu_parity_extra.py tests/test_gpu_ops.py tests/test_gpu_backward_variants.py tests/test_gpu_configs.py -x -q 2>&1 | tail -2
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-cache-bench > gpurun_out/sc.json 2>gpurun_out/sc.err; python tools/bline.py sc < gpurun_out/sc.json
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4"
$R --workload c3 --steps 10 --warmup 3 > gpurun_out/n4_c3.json 2>gpurun_out/n4_c3.err; python tools/bline.py c3 < gpurun_out/n4_c3.json
