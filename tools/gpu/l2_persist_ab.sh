# L2 access-policy window (ara_config.l2_persist) on / off: the paper config (the window covers the
# sparse block's packed rows) and dense tables (rho = 1; the window covers the column block:
# 256 MB fp64, 128 MB fp32).  Kernel ms, interleaved.
mkdir -p gpurun_out
: > gpurun_out/l2p.jsonl
for rep in 1 2; do
for cfg in "" "--rho 1.0" "--rho 1.0 --precision f32"; do
  for l2 in "" "--l2-persist"; do
    timeout 300 python tools/prof_ara.py --steps 4 $cfg $l2 2>>gpurun_out/l2p.err | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); d['cfg']='$cfg'; print(json.dumps(d))" >> gpurun_out/l2p.jsonl
  done
done; done
python - <<'PY'
import json, collections
r = collections.defaultdict(list)
for l in open('gpurun_out/l2p.jsonl'):
    d = json.loads(l); r[(d['cfg'] or 'paper', d['l2_persist'])].append(min(d['kernel_ms'][1:]))
for k, v in sorted(r.items()): print(f"{k[0]:28s} l2_persist={k[1]!s:5s} min kernel ms {min(v):.3f}  {[round(x,3) for x in v]}")
PY
