# compute-sanitizer over tools/sanitize_flow.py (see its docstring for SAN_DRIVERS / SAN_FORMB)
mkdir -p gpurun_out/san
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_flow.py > gpurun_out/san/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -1 gpurun_out/san/memcheck.log
SAN_FORMB=flow,levels timeout 1200 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_flow.py > gpurun_out/san/synccheck.log 2>&1; echo "synccheck rc=$?"; tail -1 gpurun_out/san/synccheck.log
SAN_FORMB=chunks timeout 600 compute-sanitizer --tool synccheck python tools/sanitize_flow.py > gpurun_out/san/synccheck_chunks.log 2>&1; echo "synccheck chunks rc=$?"; grep -A2 "error detected" gpurun_out/san/synccheck_chunks.log | grep "at " | sort | uniq -c
SAN_DRIVERS=stream timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_flow.py > gpurun_out/san/racecheck.log 2>&1; echo "racecheck rc=$?"; tail -1 gpurun_out/san/racecheck.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/san/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/san/pytest.log
