mkdir -p gpurun_out
: > gpurun_out/cov.jsonl
for w in 999999 40000 36000 32000 24000 16000 0; do
  ARA_BC_SMEM_WORDS=$w timeout 300 python tools/prof_ara.py --steps 4 | python -c "import json,sys; d=json.loads(sys.stdin.read()); d['words']=$w; print(json.dumps(d))" >> gpurun_out/cov.jsonl
done
ARA_LIB_PATH=$PWD/ab/x_cbuf128_unsafe.so timeout 300 python tools/prof_ara.py --steps 4 | python -c "import json,sys; d=json.loads(sys.stdin.read()); d['words']='cbuf128'; print(json.dumps(d))" >> gpurun_out/cov.jsonl
python -c "
import json
for l in open('gpurun_out/cov.jsonl'):
    d=json.loads(l); print(d['words'], round(min(d['kernel_ms'][1:]),3))
"
