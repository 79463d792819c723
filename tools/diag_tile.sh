mkdir -p gpurun_out/diag
for t in auto 1024 1280; do
  if [ $t = auto ]; then unset TSG_TILE; else export TSG_TILE=$t; fi
  TSG_DIAG=1 timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/diag/$t.json 2> gpurun_out/diag/$t.err
  grep "tile.*slots" gpurun_out/diag/$t.err | head -2
  python -c "import json; d=json.load(open('gpurun_out/diag/$t.json')); print('$t', d['value']/1e9, d['ms_per_pass'])"
done
