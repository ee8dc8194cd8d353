timeout 2000 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/r2_gpu_tests_final.txt
cat gpurun_out/r2_gpu_tests_final.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
