mkdir -p gpurun_out
export TSG_SEGV_TRACE=1
timeout 900 python -m pytest tests/test_gpu_peer.py tests/test_gpu_api.py tests/test_capi_symbols.py -x -q > gpurun_out/pytest_c7.log 2>&1; echo pytest_rc=$?; tail -30 gpurun_out/pytest_c7.log
