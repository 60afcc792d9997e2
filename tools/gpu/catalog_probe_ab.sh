# Cost of the occupancy probes that miss shared memory: the paper config at catalogues whose
# bitmap fits shared memory entirely (<= ~1.3M events) vs the paper's 2M (35 % of probes via L1/L2).
mkdir -p gpurun_out
: > gpurun_out/catalog_ab.jsonl
for rep in 1 2; do
for C in 1000000 1300000 1600000 2000000 3000000; do
  timeout 300 python tools/prof_ara.py --steps 4 --catalog $C 2>>gpurun_out/catalog_ab.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); d['catalog']=$C; print(json.dumps(d))" >> gpurun_out/catalog_ab.jsonl
done; done
python - <<'PY'
import json, collections
r = collections.defaultdict(list)
for l in open('gpurun_out/catalog_ab.jsonl'):
    d = json.loads(l); r[d['catalog']].append(min(d['kernel_ms'][1:]))
for c, v in sorted(r.items()): print(c, 'min kernel ms', round(min(v), 3), v)
PY
