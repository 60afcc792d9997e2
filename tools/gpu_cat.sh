P="python tools/prof_ara.py --steps 3"
for c in 2000000 1000000 500000 250000; do
  ARA_KERNEL=5 timeout 300 $P --catalog $c 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['catalog'], [round(x,3) for x in d['kernel_ms']])"
  ARA_KERNEL=8 timeout 300 $P --catalog $c 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tma', d['catalog'], [round(x,3) for x in d['kernel_ms']])"
done
