timeout 2200 python -m pytest tests -m gpu -q 2>&1 | tail -2 > gpurun_out/r2_gpu_tests_final.txt; cat gpurun_out/r2_gpu_tests_final.txt
for w in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $w --master-addr 127.0.0.1 --master-port 2963$w tests/dist_parity.py > gpurun_out/r2_dist_parity_w$w.txt 2>&1; echo "w$w rc=$?"; grep dist_parity gpurun_out/r2_dist_parity_w$w.txt
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
