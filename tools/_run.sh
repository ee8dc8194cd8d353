timeout 600 python -m pytest tests/test_gpu_bucket.py tests/test_gpu_parity_extra.py -x -q 2>&1 | tail -3
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-cache-bench"
$B > gpurun_out/sc.json 2>gpurun_out/sc.err; python tools/bline.py sc < gpurun_out/sc.json
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'bkt_rows' -c 3 --csv --log-file gpurun_out/l_rows.csv python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --no-cache-bench > /dev/null 2>&1
python tools/launches.py gpurun_out/l_rows.csv 2>&1 | tail -2
