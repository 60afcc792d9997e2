# metrics timing A/B over ab/*.so builds (SLOT=metrics variants) and grid sizes (ARA_METRICS_BLOCKS)
mkdir -p gpurun_out
: > gpurun_out/met_ab.jsonl
LIBS="$(ls $PWD/ab/*.so 2>/dev/null) $PWD/paper_1606_04473_b200/libara.so"
for rep in 1 2; do for lib in $LIBS; do for b in ${BLOCKS:-1 2}; do
  ARA_LIB_PATH=$lib ARA_METRICS_BLOCKS=$b timeout 300 python tools/prof_ara.py --steps 5 2>> gpurun_out/met_ab.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); d['lib']='$(basename $lib .so)'; print(json.dumps(d))" >> gpurun_out/met_ab.jsonl
done; done; done
python - <<'P'
import json, collections
r = collections.defaultdict(list)
for l in open('gpurun_out/met_ab.jsonl'):
    d = json.loads(l); r[(d['lib'], d['env'].get('ARA_METRICS_BLOCKS'))].append(min(d['metrics_ms'][1:]))
for k, v in sorted(r.items()): print(k, round(min(v), 4), [round(x, 4) for x in v])
P
