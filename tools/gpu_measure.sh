#!/bin/bash
# Round measurement pass: every BASELINE config's bench line, the c4 launch list (ncu
# gpu__time_duration), --set full captures of the round kernels and the evaluator's
# tensor-core SYRK.  Logs under gpurun_out/.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python build.py > gpurun_out/build.log 2>&1
for spec in "c4" "c4 --variant fast_alpha_fd" "c4 --variant hashing" "c4 --variant osnap" "c1" "c2" "c2 --shards 8" "c3" "c3 --ell 50" "c3 --ell 200" "c5"; do
  name=$(echo $spec | tr ' ' '_' | tr -d '-')
  timeout 900 python bench.py --workload $spec --steps 5 --warmup 3 > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
echo "ncu launch rc=$?" >> gpurun_out/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:trd_kernel|eig_kernel|bt_kernel|gram_tc|recon_i8" \
  -s 56 -c 6 -o gpurun_out/c4_full python tools/prof_c4.py > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full.log
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:syrk_i8|quant_kernel|colmax|lanczos" \
  -s 4 -c 4 -o gpurun_out/eval_full python tools/eval_time.py > gpurun_out/ncu_eval.log 2>&1
echo "ncu eval rc=$?" >> gpurun_out/ncu_eval.log
