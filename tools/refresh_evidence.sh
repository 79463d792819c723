#!/bin/bash
# Refreshes the committed evidence for the bench workload (run through gpurun, 1 GPU):
#   the default bench line, the ncu launch list + one --set full capture of tile_update
#   (tools/profile_cfg3.sh), and the one-pass timeline of a TSG_TRACE build (if built as
#   paper_1502_00355_b200/libtsg_trace.so).   usage: tools/refresh_evidence.sh TAG
set -u
TAG=$1
mkdir -p gpurun_out
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"
bash tools/profile_cfg3.sh $TAG tile_update
if [ -f paper_1502_00355_b200/libtsg_trace.so ]; then
  TSG_LIB=$PWD/paper_1502_00355_b200/libtsg_trace.so python tools/trace_cfg3.py > gpurun_out/${TAG}_timeline.txt 2>&1
fi
ncu -i gpurun_out/${TAG}_kernel.ncu-rep --page raw --csv > gpurun_out/${TAG}_kernel_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_kernel.ncu-rep --page source --csv > gpurun_out/${TAG}_kernel_source.csv 2>/dev/null
echo done
