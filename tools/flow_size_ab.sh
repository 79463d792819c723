# dataflow launch vs per-pass graph on random Delaunay meshes of growing size (calibrates kFlowWaves)
for n in 2000000 4000000 8000000; do
  for mode in graph flow; do
    if [ $mode = flow ]; then e="TSG_FORMA_FLOW=1 TSG_TILE=1280"; else e="TSG_FORMA_FLOW=0"; fi
    env $e timeout 900 python bench.py --config cfg2 --nodes $n --steps 10 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$n $mode', round(d['value']/1e9,2), round(d['ms_per_pass'],4), d['impl_config']['driver'][:10])"
  done
done
