python bench.py > gpurun_out/r2_final_n1.json 2>gpurun_out/r2_final_n1.err; python tools/bline.py final < gpurun_out/r2_final_n1.json
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'bkt|tbe' -c 60 --csv --log-file gpurun_out/r2_launches_final.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-cache-bench > /dev/null 2>&1
python tools/launches.py gpurun_out/r2_launches_final.csv | head -16
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_final_ref.json 2>gpurun_out/r2_final_ref.err; tail -c 600 gpurun_out/r2_final_ref.json
