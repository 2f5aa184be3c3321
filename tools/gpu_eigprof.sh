#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 300 python tools/debug_eigtime.py 148000 > gpurun_out/eigtime.log 2>&1
echo "rc=$?" >> gpurun_out/eigtime.log
timeout 300 python tools/prof_eig.py > gpurun_out/prof_eig_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:eig_kernel -s 2 -c 1 \
  -o gpurun_out/eig_full python tools/prof_eig.py > gpurun_out/ncu_eig.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_eig.log
