#!/bin/bash
# A/B of the trd head's tile-to-warp map (balanced default vs -DFD_TRD_FLATMAP row-major), c4 bench
# per-kernel ms, then the trd-sized parity tests on the default build
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for flags in "-DFD_TRD_FLATMAP" ""; do
  FD_NVCC_EXTRA="$flags" python build.py > /dev/null 2>&1
  echo "=== [$flags] $(cat paper_1501_06561_b200/libfd.so.flags)"
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['ms_per_step'], d['roofline']['per_kernel_ms_per_step'])"
done 2>&1 | tee gpurun_out/ab_trdmap.log
timeout 1200 python -m pytest tests -q -m gpu -x -k "c4 or c3 or int8 or golden or c2_batched" 2>&1 | tail -3 | tee -a gpurun_out/ab_trdmap.log
