mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_gpu3.log 2>&1; echo pytest_rc=$?; tail -25 gpurun_out/pytest_gpu3.log
