mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -x -q > gpurun_out/pytest_c4.log 2>&1; echo pytest_rc=$?; tail -15 gpurun_out/pytest_c4.log
for sch in flow chunks; do
timeout 300 python bench.py --config cfg1 --steps 5 --formb-schedule $sch --no-cpu-baseline > gpurun_out/b_cfg1_$sch.json 2> gpurun_out/b_cfg1_$sch.err; echo rc=$?; python -c "
import json; d=json.load(open('gpurun_out/b_cfg1_$sch.json')); print('$sch', d['value'], d['ms_per_step'], d['impl_config'])"; tail -2 gpurun_out/b_cfg1_$sch.err
done
timeout 300 python bench.py --config cfg1 --steps 5 > gpurun_out/b_cfg1.json 2> gpurun_out/b_cfg1.err; python -c "
import json; d=json.load(open('gpurun_out/b_cfg1.json')); print(d['value'], d['check'], d['cpu_baseline'])"
for sch in flow chunks levels; do
timeout 600 python bench.py --config cfg2 --form b --chunks 148 --steps 3 --formb-schedule $sch --no-cpu-baseline > gpurun_out/b_cfg2b_$sch.json 2> gpurun_out/b_cfg2b_$sch.err; python -c "
import json; d=json.load(open('gpurun_out/b_cfg2b_$sch.json')); print('cfg2 B148 $sch', d['value'], d['ms_per_pass'])"; tail -2 gpurun_out/b_cfg2b_$sch.err
done
timeout 900 python bench.py --config cfg3 --form b --chunks 148 --steps 2 --warmup 1 --passes 20 --formb-schedule flow --no-cpu-baseline > gpurun_out/b_cfg3b_flow.json 2> gpurun_out/b_cfg3b_flow.err; python -c "
import json; d=json.load(open('gpurun_out/b_cfg3b_flow.json')); print('cfg3 B148 flow', d['value'], d['ms_per_pass'])"; tail -2 gpurun_out/b_cfg3b_flow.err
