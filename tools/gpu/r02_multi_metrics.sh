# Metrics graph cache (two entries: consecutive multi-GPU runs alternate global-YLT buffers):
# the multi-GPU and metrics tests, then weak/strong lines.  Short timeouts.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 420 python -m pytest tests/test_multigpu.py tests/test_assembly_metrics_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_mm_n$N.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_mm_n$N.log
B="bench.py --steps 30 --no-e2e --no-cpu-baseline"
run() { local name=$1; shift; timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
        --master-addr 127.0.0.1 --master-port $((29850 + RANDOM % 100)) $B --gpus $N "$@" > gpurun_out/mm_$name.json 2> gpurun_out/mm_$name.err; }
run weak
run strong --scaling strong
tail -3 gpurun_out/pytest_mm_n$N.log
for f in gpurun_out/mm_*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);b=d['breakdown_ms'];print('$f',d['n_gpus'],d['scaling'],round(d['ms_per_step'],3),round(d['value']/1e6,1),'kernel',round(b['ara_kernel'],3),'met',round(b['metrics'],3),b['calls'])"; done
