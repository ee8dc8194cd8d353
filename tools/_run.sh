free -g; nproc; cat /sys/fs/cgroup/memory.max 2>/dev/null
ncu --set full --import-source on --clock-control none -k regex:'bkt_scatter|bkt_wsort' -s 2 -c 2 -o gpurun_out/r2_sc2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-cache-bench > gpurun_out/ncu_sc2.log 2>&1
tail -3 gpurun_out/ncu_sc2.log
