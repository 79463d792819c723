mkdir -p gpurun_out
TSG_SEGV_TRACE=1 timeout 300 python -m pytest tests/test_gpu_api.py -x -q -k concurrent > gpurun_out/pytest_conc.log 2>&1; echo conc_rc=$?; grep -v "^  File\|^Extension" gpurun_out/pytest_conc.log | tail -40
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_c5.log 2>&1; echo pytest_rc=$?; tail -5 gpurun_out/pytest_c5.log
for cfg in "cfg1" "cfg2 --form b --chunks 148 --steps 3" "cfg2 --form b --chunks 1 --steps 2 --passes 10"; do
set -- $cfg
timeout 300 python bench.py --config $cfg --formb-schedule flow --no-cpu-baseline > gpurun_out/b5.json 2> gpurun_out/b5.err; python -c "
import json; d=json.load(open('gpurun_out/b5.json')); print('$cfg flow', d['value'], d['ms_per_pass'])"; tail -1 gpurun_out/b5.err
done
timeout 300 python bench.py --config cfg2 --form b --chunks 1 --steps 2 --passes 10 --formb-schedule chunks --no-cpu-baseline > gpurun_out/b5.json 2> gpurun_out/b5.err; python -c "
import json; d=json.load(open('gpurun_out/b5.json')); print('cfg2 serial chunks', d['value'], d['ms_per_pass'])"
