# cfg5 (256M-node random Delaunay, fp32, to convergence) on one B200, with memory sampling and
# the sampled lockstep parity check (bench check object)
mkdir -p gpurun_out/r02
( while true; do free -g | awk 'NR==2{print "mem used", $3, "GB"}'; nvidia-smi --query-gpu=memory.used --format=csv,noheader; sleep 30; done ) > gpurun_out/r02/cfg5_mem.log 2>&1 &
MON=$!
timeout 2400 python bench.py --config cfg5 --steps 3 --warmup 3 > gpurun_out/r02/bench_cfg5.json 2> gpurun_out/r02/bench_cfg5.err; echo rc=$?
kill $MON
python -c "
import json; d=json.load(open('gpurun_out/r02/bench_cfg5.json')); print(d['value'], d['ms_per_pass'], d['roofline']['frac'], d['e2e']['value'], d['prep_split']); print(d['check'])"
tail -3 gpurun_out/r02/bench_cfg5.err; sort -k3 -n gpurun_out/r02/cfg5_mem.log | tail -2
