#!/bin/bash
# bt W1 8x4 tiles + hash mode A/B: c4 bench, hash bench per mode, full GPU tests
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python build.py > gpurun_out/build3.log 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/b3_c4.json 2> gpurun_out/b3_c4.err
for m in 0 1 2 3; do
  for v in hashing osnap; do
    FD_HASH_MODE=$m timeout 300 python bench.py --variant $v --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/b3_${v}_$m.json 2> gpurun_out/b3_${v}_$m.err
  done
done
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest3.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest3.log
