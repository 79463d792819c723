# A/B of slots per tile (TSG_TILE, compile-time sizes 768/1024/1280) plus the tests covering them
mkdir -p gpurun_out/tile3
export TSG_SEGV_TRACE=1
timeout 900 python -m pytest tests/test_gpu_layout.py tests/test_gpu_parity.py -q -x > gpurun_out/tile3/pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/tile3/pytest.log
timeout 900 python -m pytest tests/test_gpu_scale.py -q -x -k "cfg2" > gpurun_out/tile3/pytest_scale.log 2>&1; echo scale_rc=$?; tail -3 gpurun_out/tile3/pytest_scale.log
b() { tag=$1; shift; timeout 600 python bench.py --no-cpu-baseline "$@" > gpurun_out/tile3/$tag.json 2> gpurun_out/tile3/$tag.err; python -c "
import json; d=json.load(open('gpurun_out/tile3/$tag.json')); print('$tag', round(d['value']/1e9,2), 'G', round(d['ms_per_pass'],4), 'ms/pass frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']/1e9,2))" 2>&1 | tail -1; }
TSG_LIB=paper_1502_00355_b200/libtsg_head.so b cfg3_head --steps 10
for r in 1 2; do for t in 768 1024 1280; do TSG_TILE=$t b cfg3_t${t}_$r --steps 10; done; done
for t in 768 1024 1280; do TSG_TILE=$t b cfg2_t${t} --config cfg2 --steps 20; done
for t in 768 1024 1280; do TSG_TILE=$t b cfg2_f32_t${t} --config cfg2 --precision f32 --steps 20; done
for t in 1024 1280; do TSG_TILE=$t b cfg3_f32_t$t --precision f32 --steps 10; done
for t in 1024 1280; do TSG_TILE=$t b cfg4_t$t --config cfg4 --steps 3; done
TSG_LIB=paper_1502_00355_b200/libtsg_head.so b cfg4_head --config cfg4 --steps 3
echo done
