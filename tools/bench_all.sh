#!/bin/bash
# one bench line per BASELINE config (+ variants), logs under gpurun_out/
set -x
./tools/micro/peaks > gpurun_out/peaks.json 2> gpurun_out/peaks.err
for spec in "c1" "c2" "c2 --shards 8" "c3" "c3 --ell 50" "c3 --ell 200" "c4" "c4 --variant fast_alpha_fd" "c5"; do
  name=$(echo $spec | tr ' ' '_' | tr -d '-')
  timeout 900 python bench.py --workload $spec --steps 5 --warmup 3 > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err
done
