# A/B of two builds of libara.so on one box: ab/libara_prev.so vs the in-tree build, interleaved.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_random_gpu.py -q -p no:cacheprovider -x -k "${TESTS:-packed_rows or sparse or fifo or tower or random or edge or partition or multi_window}" > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ab.log
: > gpurun_out/lib_ab.jsonl
for rep in 1 2; do
for cfg in "" "--config tower" ${EXTRA_CFG}; do
  for lib in $PWD/ab/libara_prev.so $PWD/paper_1606_04473_b200/libara.so; do
    ARA_LIB_PATH=$lib timeout 300 python tools/prof_ara.py --steps 3 $cfg | python -c "import json,sys; d=json.loads(sys.stdin.read()); d['lib']='$lib'.split('/')[-2]; print(json.dumps(d))" >> gpurun_out/lib_ab.jsonl 2>> gpurun_out/lib_ab.err
  done
done
done
tail -2 gpurun_out/pytest_ab.log
python -c "
import json
for l in open('gpurun_out/lib_ab.jsonl'):
    d=json.loads(l); print(d['lib'], d['config'], d['precision'], [round(x,3) for x in d['kernel_ms']])
"
