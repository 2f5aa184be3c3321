#!/bin/bash
# A/B of the lean eig kernel's resident CTAs per SM (c4 bench, per-kernel ms)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for c in 4 3 5; do
  FD_NVCC_EXTRA="-DFD_EIG_CTAS=$c" python build.py > /dev/null 2>&1
  echo "=== FD_EIG_CTAS=$c"
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['roofline']['per_kernel_ms_per_step'])"
done
