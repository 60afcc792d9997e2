mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
nvidia-smi topo -m > gpurun_out/topo_n$N.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_n$N.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_n$N.log
for n in 2 $N; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n bench.py --gpus $n > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n --mode fold > gpurun_out/bench_fold_n$n.json 2> gpurun_out/bench_fold_n$n.err
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 tools/stream_bench.py > gpurun_out/stream_n$N.json 2> gpurun_out/stream_n$N.err
tail -2 gpurun_out/pytest_n$N.log
for f in gpurun_out/bench_n*.json gpurun_out/bench_fold_n*.json gpurun_out/stream_n$N.json; do echo $f; head -c 400 $f; echo; done
