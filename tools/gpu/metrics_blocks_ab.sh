mkdir -p gpurun_out; : > gpurun_out/mb.txt
for b in 1 2 4 8; do
  ARA_METRICS_BLOCKS=$b timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/mb_$b.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/mb_$b.json'));b=d['breakdown_ms'];print('blocks $b', round(d['ms_per_step'],3), 'metrics', round(b['metrics'],4), 'load_elts', round(b['calls']['load_elts'],4), 'kernel', round(b['ara_kernel'],3))" >> gpurun_out/mb.txt
done
cat gpurun_out/mb.txt
