# round-2 evidence (final build): GPU suite, smoke, the BASELINE config matrix, ncu captures
mkdir -p gpurun_out/r02
export TSG_SEGV_TRACE=1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/r02/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/smoke.log 2>&1; echo smoke_rc=$?
bash tools/final_bench.sh
for f in gpurun_out/r02f/bench_*.json; do cp $f gpurun_out/r02/; done
bash tools/profile_cfg3.sh r02_cfg3 tile_update
python tools/launches.py gpurun_out/r02_cfg3_launches.csv > gpurun_out/r02/cfg3_launches.txt
ncu --set full --clock-control none --import-source on -k regex:tile_flow -s 1 -c 1 -o gpurun_out/r02_cfg2_flow -f python bench.py --config cfg2 --profile --passes 20 > gpurun_out/r02/cfg2_flow_full.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02/cfg2_launches.csv python bench.py --config cfg2 --profile --passes 20 > /dev/null 2>&1
python tools/launches.py gpurun_out/r02/cfg2_launches.csv > gpurun_out/r02/cfg2_launches.txt
ncu --set full --clock-control none --import-source on -k regex:formb_flow -s 1 -c 1 -o gpurun_out/r02_cfg1_flow -f python bench.py --config cfg1 --profile > gpurun_out/r02/cfg1_flow_full.log 2>&1
head -8 gpurun_out/r02/cfg3_launches.txt
echo done
