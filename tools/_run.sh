python bench.py > gpurun_out/r2_final_n1.json 2>gpurun_out/r2_final_n1.err; python tools/bline.py final < gpurun_out/r2_final_n1.json
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'bkt|tbe' -c 60 --csv --log-file gpurun_out/r2_launches_final.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-cache-bench > /dev/null 2>&1
python tools/launches.py gpurun_out/r2_launches_final.csv | head -16
ncu --set full --import-source on --clock-control none -k regex:'bkt_rows_kernel|bkt_scatter' -c 2 -o gpurun_out/r2_final_kern python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-cache-bench > gpurun_out/ncu_final.log 2>&1
tail -1 gpurun_out/ncu_final.log
