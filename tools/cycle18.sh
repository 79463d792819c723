mkdir -p gpurun_out
export TSG_SEGV_TRACE=1
timeout 900 python -m pytest tests/test_gpu_layout.py -x -q > gpurun_out/pytest_c18a.log 2>&1; echo layout_rc=$?; tail -15 gpurun_out/pytest_c18a.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_c18.log 2>&1; echo pytest_rc=$?; tail -5 gpurun_out/pytest_c18.log
timeout 900 python bench.py --steps 10 > gpurun_out/b18_cfg3.json 2> gpurun_out/b18_cfg3.err; python -c "
import json; d=json.load(open('gpurun_out/b18_cfg3.json')); print('cfg3', d['value']/1e9, d['ms_per_pass'], d['roofline']['frac'], d['check']['match'], d['prep_s'], d['prep_split'])"
for v in default tile512; do
if [ $v = default ]; then unset TSG_LIB; else export TSG_LIB=paper_1502_00355_b200/libtsg_$v.so; fi
for cfg in cfg2 cfg3; do
timeout 600 python bench.py --config $cfg --steps 10 --no-cpu-baseline > gpurun_out/b18.json 2> gpurun_out/b18.err; python -c "
import json; d=json.load(open('gpurun_out/b18.json')); print('$v $cfg', d['value']/1e9, d['ms_per_pass'], d['roofline']['frac'])"
done
done
unset TSG_LIB
TSG_FLOW_WARP=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "flow or form_b or golden" > gpurun_out/pytest_c18b.log 2>&1; echo flow_thread_rc=$?; tail -2 gpurun_out/pytest_c18b.log
for w in 1 0; do
TSG_FLOW_WARP=$w timeout 600 python bench.py --config cfg1 --steps 10 --no-cpu-baseline > gpurun_out/b18.json 2> gpurun_out/b18.err; python -c "
import json; d=json.load(open('gpurun_out/b18.json')); print('flow_warp=$w cfg1', d['value']/1e6, 'M/s', d['ms_per_pass'])"
TSG_FLOW_WARP=$w timeout 600 python bench.py --config cfg2 --form b --chunks 1 --formb-schedule flow --steps 3 --passes 20 --no-cpu-baseline > gpurun_out/b18.json 2> gpurun_out/b18.err; python -c "
import json; d=json.load(open('gpurun_out/b18.json')); print('flow_warp=$w cfg2 serial flow', d['value']/1e9, 'G/s', d['ms_per_pass'])"
TSG_FLOW_WARP=$w timeout 600 python bench.py --config cfg2 --form b --chunks 148 --formb-schedule flow --steps 3 --passes 20 --no-cpu-baseline > gpurun_out/b18.json 2> gpurun_out/b18.err; python -c "
import json; d=json.load(open('gpurun_out/b18.json')); print('flow_warp=$w cfg2 W148 flow', d['value']/1e9, 'G/s', d['ms_per_pass'])"
done
