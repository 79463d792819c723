mkdir -p gpurun_out
export TSG_SEGV_TRACE=1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_c13.log 2>&1; echo pytest_rc=$?; tail -4 gpurun_out/pytest_c13.log
for e in X=1 TSG_NO_FUSED_FINALIZE=1; do
env $e timeout 600 python bench.py --config cfg2 --steps 10 --no-cpu-baseline > gpurun_out/b13.json 2> gpurun_out/b13.err; python -c "
import json; d=json.load(open('gpurun_out/b13.json')); print('cfg2 $e', d['value']/1e9, d['ms_per_pass'], d['roofline']['frac'], d['launches_per_step'])"
done
