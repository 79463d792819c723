mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -3 gpurun_out/smoke.log
timeout 1500 python -m pytest tests/test_gpu_scale.py -x -q --durations=20 > gpurun_out/pytest_scale.log 2>&1; echo scale_rc=$?; tail -30 gpurun_out/pytest_scale.log
timeout 900 python bench.py --steps 5 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo bench_rc=$?; python -c "
import json; d=json.load(open('gpurun_out/bench2.json')); print(d['value'], d['roofline']['frac'], d['check'], d['cpu_baseline'])"; tail -3 gpurun_out/bench2.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref2.json 2> gpurun_out/ref2.err; echo ref_rc=$?; cut -c1-300 gpurun_out/ref2.json; python -c "
import json; d=json.load(open('gpurun_out/ref2.json')); print(d['check'])"
