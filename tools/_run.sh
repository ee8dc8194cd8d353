ncu --set full --import-source on --clock-control none -k regex:'bkt_wsort' -s 1 -c 1 -o gpurun_out/r2_ws3 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-cache-bench > gpurun_out/ncu_ws3.log 2>&1
tail -2 gpurun_out/ncu_ws3.log
