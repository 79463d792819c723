# Form A tile_flow: GPU suite, then the bench with TSG_FORMA_FLOW=0/1 on cfg2
mkdir -p gpurun_out/flow2
export TSG_SEGV_TRACE=1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/flow2/pytest.log 2>&1; echo pytest_rc=$?; tail -15 gpurun_out/flow2/pytest.log
b() { tag=$1; shift; timeout 600 python bench.py "$@" > gpurun_out/flow2/$tag.json 2> gpurun_out/flow2/$tag.err; python -c "
import json; d=json.load(open('gpurun_out/flow2/$tag.json')); c=d.get('check') or {}; print('%-22s %6.2f G %.4f ms/pass frac %.3f e2e %.2f match %s %s' % ('$tag', d['value']/1e9, d['ms_per_pass'], d['roofline']['frac'], d['e2e']['value']/1e9, c.get('match'), d['impl_config']['driver'][:12]))" 2>&1 | tail -1; }
b cfg2_auto --config cfg2 --steps 20
TSG_FORMA_FLOW=0 b cfg2_graph --config cfg2 --steps 20 --no-cpu-baseline
b cfg2_auto_f32 --config cfg2 --steps 20 --precision f32 --no-cpu-baseline
b cfg2_auto_soa --config cfg2 --steps 20 --layout soa --no-cpu-baseline
b cfg3_auto --steps 10 --no-cpu-baseline
echo done
