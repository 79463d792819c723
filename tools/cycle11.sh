mkdir -p gpurun_out
export TSG_SEGV_TRACE=1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_c11.log 2>&1; echo pytest_rc=$?; tail -15 gpurun_out/pytest_c11.log
for rep in 1 2; do
for v in default f64filter; do
if [ $v = default ]; then unset TSG_LIB; else export TSG_LIB=paper_1502_00355_b200/libtsg_$v.so; fi
timeout 600 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/b11_$v.json 2> gpurun_out/b11_$v.err; python -c "
import json; d=json.load(open('gpurun_out/b11_$v.json')); print('$v', d['value']/1e9, d['ms_per_pass'], d['roofline']['frac'], d['roofline']['launch_ms_stream_driver'], d['e2e']['value']/1e9)"
done
done
unset TSG_LIB
TSG_DIAG=1 timeout 600 python bench.py --profile 2>&1 | grep "tsg diag" | awk 'NR%10==1' | head -12
