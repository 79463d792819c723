mkdir -p gpurun_out
timeout 600 python bench.py --config cfg2 --steps 10 --no-cpu-baseline > gpurun_out/b12_cfg2.json 2> gpurun_out/b12_cfg2.err; python -c "
import json; d=json.load(open('gpurun_out/b12_cfg2.json')); print('cfg2', d['value']/1e9, d['ms_per_pass'], d['roofline']['frac'], d['roofline']['launch_ms_stream_driver'], d['launches_per_step'])"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -c 40 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --config cfg2 --profile --passes 10 > /dev/null 2>&1; python tools/launches.py gpurun_out/launches_cfg2.csv | tail -25
