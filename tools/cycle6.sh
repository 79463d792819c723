mkdir -p gpurun_out
export TSG_SEGV_TRACE=1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_c6.log 2>&1; echo pytest_rc=$?; grep -v "^  File\|^Extension" gpurun_out/pytest_c6.log | tail -30
timeout 300 python bench.py --config cfg1 --steps 10 > gpurun_out/b6_cfg1.json 2> gpurun_out/b6_cfg1.err; python -c "
import json; d=json.load(open('gpurun_out/b6_cfg1.json')); print('cfg1', d['value'], d['ms_per_pass'], d['check']['match'], d['cpu_baseline']['value'])"; grep "Form B" gpurun_out/b6_cfg1.err
TSG_DIAG=1 timeout 300 python bench.py --config cfg2 --form b --chunks 148 --steps 2 --no-cpu-baseline --passes 20 2>&1 >/dev/null | grep "Form B"
TSG_DIAG=1 timeout 300 python bench.py --config cfg2 --form b --chunks 1 --steps 2 --no-cpu-baseline --passes 20 > gpurun_out/b6_cfg2s.json 2> gpurun_out/b6_cfg2s.err; grep "Form B" gpurun_out/b6_cfg2s.err; python -c "
import json; d=json.load(open('gpurun_out/b6_cfg2s.json')); print('cfg2 serial auto', d['value'], d['ms_per_pass'])"
