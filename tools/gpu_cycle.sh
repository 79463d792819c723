mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -5 gpurun_out/pytest_gpu.log
python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?; cut -c1-400 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --profile --passes 6 > /dev/null 2>&1; python tools/launches.py gpurun_out/launches.csv
TSG_DIAG=1 python bench.py --profile 2>&1 | grep "tsg diag" | awk "NR%10==1"
