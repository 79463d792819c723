# A/B of an environment switch on the default bench (usage: tools/ab.sh VAR=1)
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for e in "X=1" "$@"; do env $e python bench.py --no-cpu-baseline --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$e\", d[\"value\"]/1e9, d[\"ms_per_pass\"], d['e2e']['value']/1e9)"; done
