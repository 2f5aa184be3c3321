#!/bin/bash
# ncu --set full of the Hashing (s = 1) and OSNAP (s = 4) kernels at c4 (one launch each)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python build.py > gpurun_out/build.log 2>&1
for v in hashing osnap; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:hash_kernel|hash_reduce" -s 2 -c 2 \
    -o gpurun_out/hash_$v -f python bench.py --variant $v --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_hash_$v.log 2>&1
  echo "ncu $v rc=$?" >> gpurun_out/ncu_hash_$v.log
done
