mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt; nproc >> gpurun_out/smi.txt; free -g >> gpurun_out/smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?; cut -c1-600 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
