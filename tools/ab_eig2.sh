#!/bin/bash
# A/B of the lean eig kernel's resident CTAs per SM after the fp32 inverse-iteration scratch
# (c4 bench, per-kernel ms); build.py rebuilds when FD_NVCC_EXTRA changes
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for flags in "" "-DFD_EIG_CTAS=4" "-DFD_EIG_CTAS=5" "-DFD_EIG_CTAS=2"; do
  FD_NVCC_EXTRA="$flags" python build.py > /dev/null 2>&1
  echo "=== [$flags] $(cat paper_1501_06561_b200/libfd.so.flags)"
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['roofline']['per_kernel_ms_per_step'])"
done 2>&1 | tee gpurun_out/ab_eig2.log
python build.py > /dev/null 2>&1
