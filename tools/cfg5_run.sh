# cfg5 (256M-node random Delaunay, fp32, to convergence) on one B200, with memory sampling
mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests/test_gpu_layout.py -x -q > gpurun_out/r02/pytest_layout.log 2>&1; echo layout_rc=$?; tail -3 gpurun_out/r02/pytest_layout.log
( while true; do free -g | awk 'NR==2{print "mem used", $3, "GB"}'; nvidia-smi --query-gpu=memory.used --format=csv,noheader; sleep 30; done ) > gpurun_out/r02/cfg5_mem.log 2>&1 &
MON=$!
timeout 2400 python bench.py --config cfg5 --steps 1 --warmup 1 > gpurun_out/r02/bench_cfg5.json 2> gpurun_out/r02/bench_cfg5.err; echo rc=$?
kill $MON
cut -c1-2500 gpurun_out/r02/bench_cfg5.json; tail -20 gpurun_out/r02/bench_cfg5.err; sort -k3 -n gpurun_out/r02/cfg5_mem.log | tail -3
