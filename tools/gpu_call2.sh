#!/bin/bash
# hash ILP check (parity + bench), tf32 operand-conversion microtest, bt/eig source-level capture
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python build.py > gpurun_out/build2.log 2>&1
./tools/micro/tf32_conv > gpurun_out/tf32_conv.txt 2>&1
timeout 600 python -m pytest tests -q -m gpu -k "hash" > gpurun_out/pytest_hash.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_hash.log
for v in hashing osnap; do
  timeout 600 python bench.py --variant $v --steps 5 --warmup 3 > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:bt_kernel|eig_kernel" \
  -s 40 -c 2 -o gpurun_out/bt_eig python tools/prof_c4.py > gpurun_out/ncu_bteig.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_bteig.log
