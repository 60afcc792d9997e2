# A/B of several builds of libara.so on one box: every ab/*.so (plus the
# in-tree build as "tree"): oracle checks (tests/gpu_check_bc.py), then timings
# interleaved over REPS rounds.  EXTRA_CFG: more prof_ara.py argument sets,
# separated by ';' (e.g. "--config tower;--precision f32").
mkdir -p gpurun_out
: > gpurun_out/ab.jsonl
: > gpurun_out/ab_summary.txt
LIBS="$(ls $PWD/ab/*.so 2>/dev/null) $PWD/paper_1606_04473_b200/libara.so"
for lib in $LIBS; do
  n=$(basename $(dirname $lib))_$(basename $lib .so)
  ARA_LIB_PATH=$lib timeout 400 python tests/gpu_check_bc.py 30 > gpurun_out/ab_check_$n.log 2>&1
  echo "$n check rc=$? $(tail -1 gpurun_out/ab_check_$n.log)" >> gpurun_out/ab_summary.txt
done
IFS=';' read -ra CFGS <<< "${EXTRA_CFG:-}"
for rep in $(seq ${REPS:-3}); do
  for lib in $LIBS; do
    n=$(basename $(dirname $lib))_$(basename $lib .so)
    for cfg in "" "${CFGS[@]}"; do
      ARA_LIB_PATH=$lib timeout 300 python tools/prof_ara.py --steps 4 $cfg 2>> gpurun_out/ab.err | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); d['lib']='$n'; d['cfg']='$cfg'; print(json.dumps(d))" >> gpurun_out/ab.jsonl
    done
  done
done
python - <<'PY' >> gpurun_out/ab_summary.txt
import json, collections
r = collections.defaultdict(list)
for l in open('gpurun_out/ab.jsonl'):
    d = json.loads(l); r[(d['cfg'], d['lib'])].append(min(d['kernel_ms'][1:]))
for (cfg, lib), v in sorted(r.items()):
    print(f"{cfg or 'paper':28s} {lib:24s} min {min(v):.3f} ms  all {[round(x, 3) for x in v]}")
PY
cat gpurun_out/ab_summary.txt
