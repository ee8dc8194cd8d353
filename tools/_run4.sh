timeout 1200 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_bytes.py tests/test_gpu_dist.py tests/test_gpu_ops.py -x -q 2>&1 | tail -4
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4"
for w in c5 c3; do
  $R --workload $w --steps 12 --warmup 3 > gpurun_out/n4_${w}.json 2>gpurun_out/n4_${w}.err; python tools/bline.py $w < gpurun_out/n4_${w}.json
  python - <<PY
import json
d=json.loads([l for l in open("gpurun_out/n4_${w}.json") if l.startswith("{")][-1])
print(d["phases_ms"], d.get("e2e",{}).get("ms_per_step"), d.get("alltoall_nvlink",{}).get("busbw_gbs"), d["alltoall"]["busbw_gbs"])
PY
done
