# A/B of experiment libraries (tools/build_variant.sh) on bench configs, alternating, same box.
# usage: tools/lib_ab.sh OUTDIR "lib1 lib2 ..." "bench args; bench args; ..."   (lib "cur" = libtsg.so)
out=gpurun_out/$1; libs=$2; IFS=';' read -ra cfgs <<< "$3"
mkdir -p $out
for r in 1 2; do for c in "${cfgs[@]}"; do for l in $libs; do
  if [ "$l" = cur ]; then lp=""; else lp=paper_1502_00355_b200/libtsg_$l.so; fi
  tag=$(echo "$c" | tr -d ' -' | tr '/' '_')_${l}_$r
  TSG_LIB=$lp timeout 600 python bench.py --no-cpu-baseline $c > $out/$tag.json 2> $out/$tag.err
  python -c "
import json; d=json.load(open('$out/$tag.json')); print('%-40s %6.2f G %.4f ms/pass frac %.3f' % ('$tag', d['value']/1e9, d['ms_per_pass'], d['roofline']['frac']))" 2>&1 | tail -1
done; done; done
