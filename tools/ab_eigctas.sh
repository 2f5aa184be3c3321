#!/bin/bash
# A/B of eig build flags (c4 bench, per-kernel ms); build.py rebuilds when FD_NVCC_EXTRA changes
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for flags in "" "-DFD_RC2_BK=32" "-DFD_RC2_STAGES=3" "-DFD_RC2_STAGES=5" "-DFD_RC2_BK=32 -DFD_RC2_STAGES=3"; do
  FD_NVCC_EXTRA="$flags" python build.py > /dev/null 2>&1
  echo "=== [$flags] $(cat paper_1501_06561_b200/libfd.so.flags)"
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['roofline']['per_kernel_ms_per_step'])"
done
python build.py > /dev/null 2>&1
