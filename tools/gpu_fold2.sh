P="python tools/prof_ara.py --steps 3"
for m in direct fold; do
  for c in paper multilayer; do
    timeout 300 $P --mode $m --config $c | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['mode'], d['config'], d['precision'], [round(x,3) for x in d['kernel_ms']])"
  done
  timeout 300 $P --mode $m --precision f32 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['mode'], d['config'], d['precision'], [round(x,3) for x in d['kernel_ms']])"
done
timeout 600 python bench.py --mode fold --no-cpu-baseline > gpurun_out/bench_fold.json 2>gpurun_out/bench_fold.err
head -c 1500 gpurun_out/bench_fold.json
