# ncu --set full of one kernel (default: the ARA trial kernel) on the paper config, after a plain run.
# usage: bash tools/gpu/ncu_kernel.sh [kernel-regex] [out-name] [extra prof_ara args]
mkdir -p gpurun_out
K=${1:-trial_kernel}; O=${2:-prof}; shift 2 2>/dev/null
Q="python tools/prof_ara.py --steps 1 $*"
timeout 300 $Q > gpurun_out/plain_q.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/$O $Q > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out/$O.ncu-rep
