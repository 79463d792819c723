mkdir -p gpurun_out
export TSG_SEGV_TRACE=1
for tr in p2p gloo; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --transport $tr --config cfg2 --nodes 200000 --passes 20 --steps 2 --warmup 1 > gpurun_out/b10_$tr.json 2> gpurun_out/b10_$tr.err; echo rc=$?
cut -c1-700 gpurun_out/b10_$tr.json; tail -3 gpurun_out/b10_$tr.err
done
