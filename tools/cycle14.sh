mkdir -p gpurun_out
for cfg in cfg2 cfg3; do
for u in 1 2 4; do
TSG_GRAPH_UNROLL=$u timeout 600 python bench.py --config $cfg --steps 10 --no-cpu-baseline > gpurun_out/b14.json 2> gpurun_out/b14.err; python -c "
import json; d=json.load(open('gpurun_out/b14.json')); print('$cfg unroll $u', d['value']/1e9, d['ms_per_pass'], d['roofline']['frac'])"
done
done
