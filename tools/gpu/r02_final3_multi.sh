# Final round-2 multi-GPU set at HEAD (run with --gpus 4): multi-GPU tests, weak/strong at N=2 and N=4
# (the default bench line per N: what the driver's scaling run executes).
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 420 python -m pytest tests/test_multigpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_multi3_n$N.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_multi3_n$N.log
run() { local name=$1 n=$2; shift 2; timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
        --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 100)) bench.py --gpus $n "$@" > gpurun_out/m3_$name.json 2> gpurun_out/m3_$name.err; }
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/m3_fw_n1.json 2> gpurun_out/m3_fw_n1.err
run fw_n2 2
run fw_n4 $N
run fs_n2 2 --scaling strong --no-cpu-baseline --no-e2e
run fs_n4 $N --scaling strong --no-cpu-baseline --no-e2e
tail -2 gpurun_out/pytest_multi3_n$N.log
for f in gpurun_out/m3_*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);b=d['breakdown_ms'];print('$f',d['n_gpus'],d['scaling'],round(d['ms_per_step'],3),round(d['value']/1e6,1),'kernel',round(b['ara_kernel'],3),'ag',round(b['allgather'],3),'met',round(b['metrics'],3),'e2e',round(d['e2e']['value']/1e6,2) if d.get('e2e') else None)"; done
