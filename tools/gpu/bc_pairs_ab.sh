# trial_kernel_bc shared-memory filter A/B: exact + pair words (default) vs
# exact words only (ARA_BC_NO_PAIRS=1, the rest probed in L1/L2); oracle checks first.
mkdir -p gpurun_out
timeout 400 python tests/gpu_check_bc.py 30 > gpurun_out/pairs_check.log 2>&1; echo "check rc=$? $(tail -1 gpurun_out/pairs_check.log)"
ARA_BC_NO_PAIRS=1 timeout 400 python tests/gpu_check_bc.py 30 > gpurun_out/pairs_check_nopairs.log 2>&1; echo "check nopairs rc=$? $(tail -1 gpurun_out/pairs_check_nopairs.log)"
: > gpurun_out/pairs_ab.jsonl
for rep in 1 2; do
  for env in "ARA_BC_NO_PAIRS=0" "ARA_BC_NO_PAIRS=1"; do
    for cfg in "" "--config tower" "--precision f32"; do
      env $env timeout 300 python tools/prof_ara.py --steps 4 $cfg | python -c "import json,sys; d=json.loads(sys.stdin.read()); d['ab']='$env'; d['cfg']='$cfg'; print(json.dumps(d))" >> gpurun_out/pairs_ab.jsonl
    done
  done
done
python -c "
import json, collections
r = collections.defaultdict(list)
for l in open('gpurun_out/pairs_ab.jsonl'):
    d = json.loads(l); r[(d['cfg'], d['ab'])].append(min(d['kernel_ms'][1:]))
for k, v in sorted(r.items()): print(f'{k[0] or \"paper\":18s} {k[1]:20s} {min(v):.3f}', [round(x,3) for x in v])
"
