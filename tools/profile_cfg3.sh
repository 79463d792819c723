#!/bin/bash
# ncu evidence for the bench workload (run on the GPU box through gpurun, 1 GPU):
#   gpurun_out/<tag>_launches.csv  per-launch duration + DRAM bytes of every kernel of a short
#                                  stream-driver smooth (cold-cache, serialised: compare shares)
#   gpurun_out/<tag>_<k>.ncu-rep   one --set full capture of kernel regex <k>
# usage: tools/profile_cfg3.sh TAG KERNEL_REGEX [bench args...]
set -u
TAG=$1; KRE=$2; shift 2
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --profile --passes 6 "$@" \
    > gpurun_out/${TAG}_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:${KRE} -s 4 -c 1 \
    -o gpurun_out/${TAG}_kernel -f python bench.py --profile --passes 6 "$@" > gpurun_out/${TAG}_full.log 2>&1
echo "profile done: $TAG"
