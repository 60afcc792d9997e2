# NVLink traffic of the fused YLT assembly (kernel-epilogue peer stores, a9) vs
# the ncclAllGather fallback at N GPUs: nvidia-smi NVLink data counters read
# before and after each run of the weak-scaling bench (K steps + warm-up).
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
snap() { nvidia-smi nvlink -gt d > "$1" 2>&1; }
run() {  # name, env...
  local name=$1; shift
  snap gpurun_out/nvl_${name}_before.txt
  env "$@" timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --steps 50 --warmup 5 --no-e2e --no-cpu-baseline \
      > gpurun_out/nvl_${name}.json 2> gpurun_out/nvl_${name}.err
  snap gpurun_out/nvl_${name}_after.txt
}
run fused ARA_DUMMY=0
run allgather ARA_NO_P2P=1
python tools/nvlink_delta.py gpurun_out/nvl_fused_before.txt gpurun_out/nvl_fused_after.txt gpurun_out/nvl_fused.json > gpurun_out/nvl_summary.txt
python tools/nvlink_delta.py gpurun_out/nvl_allgather_before.txt gpurun_out/nvl_allgather_after.txt gpurun_out/nvl_allgather.json >> gpurun_out/nvl_summary.txt
cat gpurun_out/nvl_summary.txt; head -30 gpurun_out/nvl_fused_before.txt
