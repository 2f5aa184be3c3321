#!/bin/bash
# A/B of the Hashing kernel's bucket-class count G (FD_HASH_G; 0 = one thread per column), c4, s = 1;
# then the lean eig CTAs-per-SM A/B (tools/ab_eig2.sh)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python build.py > gpurun_out/build.log 2>&1
for g in 0 2 4 8; do
  echo "=== FD_HASH_G=$g"
  FD_HASH_G=$g timeout 600 python -m pytest tests -q -m gpu -k "hash" 2>&1 | tail -1
  FD_HASH_G=$g timeout 600 python bench.py --variant hashing --steps 5 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['ms_per_step'], d['roofline'])"
done 2>&1 | tee gpurun_out/ab_hash_g.log
echo "=== osnap (unchanged kernel)" | tee -a gpurun_out/ab_hash_g.log
timeout 600 python bench.py --variant osnap --steps 5 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['ms_per_step'])" 2>&1 | tee -a gpurun_out/ab_hash_g.log
bash tools/ab_eig2.sh
