# 4 GPUs: full GPU tests (incl. sharded torchrun tests), bench at 2 and 4 GPUs, streamed 10M-trial YET.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_n$N.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_n$N.log
for n in 2 $N; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n bench.py --gpus $n --steps 20 > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29544 bench.py --gpus $N --steps 10 --config multilayer --no-cpu-baseline > gpurun_out/bench_ml_n$N.json 2> gpurun_out/bench_ml_n$N.err
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 tools/stream_bench.py > gpurun_out/stream_n$N.json 2> gpurun_out/stream_n$N.err
tail -2 gpurun_out/pytest_n$N.log
for f in gpurun_out/bench_n*.json gpurun_out/bench_ml_n$N.json; do python -c "
import json;d=json.load(open('$f'));r=d['roofline'];print('$f',d['n_gpus'],round(d['ms_per_step'],3),round(d['value']/1e6,2),'Mtrials/s k',round(r['kernel_ms'],3),'ag',round(d['breakdown_ms']['allgather'],3),'met',round(d['breakdown_ms']['metrics'],3),'e2e',round(d['e2e']['value']/1e6,2) if d.get('e2e') else None)"; done
cat gpurun_out/stream_n$N.json
