timeout 900 python -m pytest tests/test_gpu_backward_variants.py tests/test_gpu_configs.py -x -q 2>&1 | tail -1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 tools/profile_sharded.py --workload c5 --gpus 4 > gpurun_out/prof_c5c.txt 2>gpurun_out/prof_c5c.err
grep -E "hot_chunk|pipe_update|phases" gpurun_out/prof_c5c.txt
