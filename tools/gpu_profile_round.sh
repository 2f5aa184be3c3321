#!/bin/bash
# Bench line + ncu launch list of the bench command + one --set full capture per hot kernel.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r1.log 2> gpurun_out/bench_r1.err
echo "bench rc=$?" >> gpurun_out/bench_r1.err
timeout 600 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
echo "ncu launch rc=$?" >> gpurun_out/ncu_launch.log
timeout 300 python tools/prof_c4.py > gpurun_out/prof_c4_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:trd_kernel|eig_kernel|bt_kernel|gram_tc|recon|ingest" \
  -s 56 -c 7 -o gpurun_out/c4_full python tools/prof_c4.py > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full.log
