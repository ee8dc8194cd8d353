timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_sharded.py tests/test_gpu_bytes.py tests/test_gpu_configs.py tests/test_gpu_dlrm.py tests/test_gpu_dropin.py -x -q 2>&1 | tail -2
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4"
$R --workload c3 --steps 10 --warmup 3 > gpurun_out/n4_c3.json 2>gpurun_out/n4_c3.err; python tools/bline.py c3 < gpurun_out/n4_c3.json
$R --workload c5 --steps 10 --warmup 3 > gpurun_out/n4_c5.json 2>gpurun_out/n4_c5.err; python tools/bline.py c5 < gpurun_out/n4_c5.json
