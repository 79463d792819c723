# round-2 evidence (final build): GPU suite, the BASELINE config matrix, ncu captures
mkdir -p gpurun_out/r02
export TSG_SEGV_TRACE=1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/r02/pytest_gpu.log
run() { tag=$1; shift; timeout 1200 python bench.py "$@" > gpurun_out/r02/bench_$tag.json 2> gpurun_out/r02/bench_$tag.err; echo "$tag rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/r02/bench_$tag.json')); c=d.get('check') or {}; print('  ', round(d['value']/1e9,3), 'G', round(d['ms_per_pass'],4), 'ms/pass frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']/1e9,2), 'match', c.get('match'), 'cpu', (d.get('cpu_baseline') or {}).get('value'), d['impl_config']['driver'][:10], 'prep', d.get('prep_split'))" 2>&1 | tail -1; }
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
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02/bench_reference_cfg3.json 2> gpurun_out/r02/bench_reference_cfg3.err; echo ref_rc=$?; cut -c1-600 gpurun_out/r02/bench_reference_cfg3.json
bash tools/profile_cfg3.sh r02_cfg3 tile_update
python tools/launches.py gpurun_out/r02_cfg3_launches.csv > gpurun_out/r02/cfg3_launches.txt
ncu --set full --clock-control none --import-source on -k regex:tile_flow -s 1 -c 1 -o gpurun_out/r02_cfg2_flow -f python bench.py --config cfg2 --profile --passes 20 > gpurun_out/r02/cfg2_flow_full.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02/cfg2_launches.csv python bench.py --config cfg2 --profile --passes 20 > /dev/null 2>&1
python tools/launches.py gpurun_out/r02/cfg2_launches.csv > gpurun_out/r02/cfg2_launches.txt
ncu --set full --clock-control none --import-source on -k regex:formb_flow -c 1 -o gpurun_out/r02_cfg1_flow -f python bench.py --config cfg1 --profile > gpurun_out/r02/cfg1_flow_full.log 2>&1
cat gpurun_out/r02/cfg3_launches.txt gpurun_out/r02/cfg2_launches.txt
echo done
