# final-build bench lines for profiles/r02 (the configs whose numbers DESIGN/README quote)
mkdir -p gpurun_out/r02f
run() { tag=$1; shift; timeout 1200 python bench.py "$@" > gpurun_out/r02f/bench_$tag.json 2> gpurun_out/r02f/bench_$tag.err; echo "$tag rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/r02f/bench_$tag.json')); c=d.get('check') or {}; print('  ', round(d['value']/1e9,3), 'G', round(d['ms_per_pass'],4), 'ms/pass frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']/1e9,3), 'match', c.get('match'), 'cpu', (d.get('cpu_baseline') or {}).get('value'), 'prep', sum(v for k,v in d['prep_split'].items() if k.endswith('_s')), d['clocks'])" 2>&1 | tail -1; }
run cfg3_f64 --steps 10
run cfg1 --config cfg1 --steps 10
run cfg2_aos --config cfg2 --steps 20
run cfg2_soa --config cfg2 --layout soa --steps 20 --no-cpu-baseline
run cfg2_copy --config cfg2 --swap copy --steps 20 --no-cpu-baseline
run cfg2_f32 --config cfg2 --precision f32 --steps 20 --no-cpu-baseline
run cfg2_b148_aos --config cfg2 --form b --chunks 148 --steps 5
run cfg2_b148_soa --config cfg2 --form b --chunks 148 --layout soa --steps 5 --no-cpu-baseline
run cfg3_f32 --precision f32 --steps 10 --no-cpu-baseline
run cfg3_b148 --form b --chunks 148 --steps 3 --warmup 3 --passes 20 --no-cpu-baseline
run cfg4 --config cfg4 --steps 3
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02f/bench_reference_cfg3.json 2> gpurun_out/r02f/bench_reference_cfg3.err; echo ref_rc=$?

echo done
