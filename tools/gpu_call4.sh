#!/bin/bash
# hash load-batch A/B (s = 1: 32 vs 64 rows; s = 4: 16 vs 32) + hash parity tests
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python build.py > gpurun_out/build4.log 2>&1
for b in 32 64 16; do
  FD_HASH_BATCH=$b timeout 300 python bench.py --variant hashing --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/b4_hashing_$b.json 2> gpurun_out/b4_hashing_$b.err
done
for b in 16 32; do
  FD_HASH_BATCH=$b timeout 300 python bench.py --variant osnap --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/b4_osnap_$b.json 2> gpurun_out/b4_osnap_$b.err
done
FD_HASH_BATCH=64 timeout 600 python -m pytest tests -q -m gpu -k "hash" > gpurun_out/pytest4_64.log 2>&1
timeout 600 python -m pytest tests -q -m gpu -k "hash" > gpurun_out/pytest4.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest4.log
