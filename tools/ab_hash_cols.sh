#!/bin/bash
# A/B of the Hashing kernel's slice width (columns per CTA) and CTAs per SM, c4, s = 1
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for flags in "" "-DFD_HASH_COLS=128 -DFD_HASH_CTAS=1" "-DFD_HASH_COLS=96 -DFD_HASH_CTAS=2" "-DFD_HASH_COLS=32 -DFD_HASH_CTAS=6"; do
  FD_NVCC_EXTRA="$flags" python build.py > /dev/null 2>&1
  echo "=== [$flags] $(cat paper_1501_06561_b200/libfd.so.flags)"
  timeout 600 python -m pytest tests -q -m gpu -k "hash_parity" 2>&1 | tail -1
  timeout 600 python bench.py --variant hashing --steps 5 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('hashing', d['value'], d['ms_per_step'], d['roofline']['frac'])"
done 2>&1 | tee gpurun_out/ab_hash_cols.log
python build.py > /dev/null 2>&1
