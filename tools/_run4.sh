for w in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $w --master-addr 127.0.0.1 --master-port 2961$w tests/dist_parity.py > gpurun_out/r2_dist_parity_w$w.txt 2>&1; echo "w$w rc=$?"; grep dist_parity gpurun_out/r2_dist_parity_w$w.txt
done
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29521"
$R --nproc-per-node 2 bench.py --gpus 2 > gpurun_out/r2_bench_n2.json 2>gpurun_out/r2_bench_n2.err; python tools/bline.py n2 < gpurun_out/r2_bench_n2.json
$R --nproc-per-node 4 bench.py --gpus 4 > gpurun_out/r2_bench_n4_nvlink.json 2>gpurun_out/r2_bench_n4_nvlink.err; python tools/bline.py n4 < gpurun_out/r2_bench_n4_nvlink.json
