#!/bin/bash
# A/B: inverse-iteration sweeps (FD_INV_ITERS) -- accuracy vs the oracle and c4 step time
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for it in 2 1; do
  FD_NVCC_EXTRA="-DFD_INV_ITERS=$it" python build.py > /dev/null 2>&1
  echo "=== FD_INV_ITERS=$it"
  TAG="it$it" python tools/ab_err.py 2>&1 | tail -5
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bq.log 2>&1
  python -c "
import json
for l in open('gpurun_out/bq.log'):
    if l.startswith('{'):
        d=json.loads(l); print(round(d['value']), round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['roofline']['per_kernel_ms_per_step'].items()}, d['cov_err'])
"
  timeout 900 python -m pytest tests/test_gpu_golden.py -x -q -k "c3 or c2" 2>&1 | tail -2
done
FD_NVCC_EXTRA="" python build.py > /dev/null 2>&1
