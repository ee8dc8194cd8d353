set -x
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-cache-bench"
$B > gpurun_out/ov_base.json 2>gpurun_out/ov_base.err; python tools/bline.py base < gpurun_out/ov_base.json
for k in 1 2 3; do $B --overlap-sort $k > gpurun_out/ov_$k.json 2>gpurun_out/ov_$k.err; python tools/bline.py ov$k < gpurun_out/ov_$k.json; done
