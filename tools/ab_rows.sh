#!/bin/bash
# A/B the bucketed backward variants in abv/: per-kernel launch times (ncu)
for lib in default abv/libneob200_*.so; do
  if [ "$lib" = default ]; then unset NEO_B200_LIB; else export NEO_B200_LIB=$PWD/$lib; fi
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/ab_$(basename $lib .so).csv -k regex:bkt_ python bench.py --steps 1 --warmup 1 \
      --no-cpu-baseline --no-cache-bench --no-e2e > /dev/null 2>&1
  echo "== $lib"; python tools/launches.py gpurun_out/ab_$(basename $lib .so).csv | grep -E "rows|sort|scatter|scan|count"
done
