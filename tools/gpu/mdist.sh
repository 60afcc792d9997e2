# distributed metrics (F4): multi-GPU tests + weak-scaling bench with/without
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 1200 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider > gpurun_out/pytest_mg.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_mg.log
for d in 0 1; do
  ARA_METRICS_DIST=$d timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2963$d bench.py --gpus $N --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/md_$d.json 2> gpurun_out/md_$d.err
done
tail -3 gpurun_out/pytest_mg.log
for f in gpurun_out/md_*.json; do python -c "
import json;d=json.load(open('$f'));print('$f',d['n_gpus'],d['scaling'],round(d['ms_per_step'],3),round(d['value']/1e6,2),'M', d['breakdown_ms'])"; done
