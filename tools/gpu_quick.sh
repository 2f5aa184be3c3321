python build.py > /dev/null 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
for W in "--workload c4" "--workload c3 --ell 200" "--workload c3 --ell 100"; do
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e $W > gpurun_out/bq.log 2>&1
python -c "
import json
for l in open('gpurun_out/bq.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$W', round(d['value']), round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['roofline']['per_kernel_ms_per_step'].items()})
"
done
