# final cfg2 lines (dataflow launch), sanitizers on the flow kernels, GPU suite
mkdir -p gpurun_out/r02g gpurun_out/san
export TSG_SEGV_TRACE=1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02g/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/r02g/pytest_gpu.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_flow.py > gpurun_out/san/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -1 gpurun_out/san/memcheck.log
SAN_DRIVERS=stream timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_flow.py > gpurun_out/san/racecheck.log 2>&1; echo "racecheck rc=$?"; tail -1 gpurun_out/san/racecheck.log
run() { tag=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/r02g/bench_$tag.json 2> gpurun_out/r02g/bench_$tag.err; echo "$tag rc=$?"; }
run cfg2_aos --config cfg2 --steps 20
run cfg2_soa --config cfg2 --layout soa --steps 20 --no-cpu-baseline
run cfg2_copy --config cfg2 --swap copy --steps 20 --no-cpu-baseline
run cfg2_f32 --config cfg2 --precision f32 --steps 20 --no-cpu-baseline
ncu --set full --clock-control none --import-source on -k regex:tile_flow -s 1 -c 1 -o gpurun_out/r02_cfg2_flow -f python bench.py --config cfg2 --profile --passes 20 > gpurun_out/r02g/cfg2_flow_full.log 2>&1
echo done
