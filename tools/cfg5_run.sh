# cfg5 (256M-node random Delaunay, fp32, to convergence) on one B200, with memory sampling;
# then the cfg1 formb_flow capture (skipping the 2-pass probe launch of --profile)
mkdir -p gpurun_out/r02
( while true; do free -g | awk 'NR==2{print "mem used", $3, "GB"}'; nvidia-smi --query-gpu=memory.used --format=csv,noheader; sleep 30; done ) > gpurun_out/r02/cfg5_mem.log 2>&1 &
MON=$!
timeout 2400 python bench.py --config cfg5 --steps 3 --warmup 3 > gpurun_out/r02/bench_cfg5.json 2> gpurun_out/r02/bench_cfg5.err; echo rc=$?
kill $MON
cut -c1-2500 gpurun_out/r02/bench_cfg5.json; tail -5 gpurun_out/r02/bench_cfg5.err; sort -k3 -n gpurun_out/r02/cfg5_mem.log | tail -3
ncu --set full --clock-control none --import-source on -k regex:formb_flow -s 1 -c 1 -o gpurun_out/r02_cfg1_flow -f python bench.py --config cfg1 --profile > gpurun_out/r02/cfg1_flow_full.log 2>&1
echo done
