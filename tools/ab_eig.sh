#!/bin/bash
# A/B of eig build flags: stream + merge eig phase times (c4, P = 2368)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for flags in "" "-DFD_SOLVE_BATCH=4" "-DFD_PANEL_INLINE" "-DFD_PANEL_INLINE -DFD_SOLVE_BATCH=4"; do
  FD_NVCC_EXTRA="$flags" python build.py > /dev/null 2>&1
  echo "=== flags: [$flags]"
  python tools/debug_c4eig.py 2368 2>&1 | tail -2
  python tools/debug_merge_eig.py 2368 2>&1 | head -2
done
