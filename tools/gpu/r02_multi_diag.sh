# Why is the trial kernel slower at N > 1 (weak scaling, same per-rank work)?  Same box:
# N=1, N=4 default, N=4 without NVLS, N=4 without the fused peer stores, N=4 with NCCL P2P off.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
B="bench.py --steps 30 --no-e2e --no-cpu-baseline"
timeout 600 python $B > gpurun_out/diag_n1.json 2> gpurun_out/diag_n1.err
run() { local name=$1; shift; env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
        --master-addr 127.0.0.1 --master-port $((29800 + RANDOM % 150)) $B --gpus $N > gpurun_out/diag_$name.json 2> gpurun_out/diag_$name.err; }
run n4 ARA_X=0
run n4_nonvls NCCL_NVLS_ENABLE=0
run n4_nop2p ARA_NO_P2P=1
run n4_ncclp2poff NCCL_P2P_DISABLE=1 ARA_NO_P2P=1
for f in gpurun_out/diag_*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);b=d['breakdown_ms'];print('$f',d['n_gpus'],round(d['ms_per_step'],3),round(d['value']/1e6,1),'kernel',round(b['ara_kernel'],3),'ag',round(b['allgather'],3),'met',round(b['metrics'],3),b['calls'])"; done
