# One iteration check of the in-tree build: oracle checks + kernel timings (ab_libs with no A/B libs),
# the GPU test suite, and an ncu --set full capture of the sparse trial kernel with its hot SASS lines.
mkdir -p gpurun_out
REPS=2 EXTRA_CFG="--config tower;--precision f32" timeout 900 bash tools/gpu/ab_libs.sh > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 bash tools/gpu/ncu_kernel.sh trial_kernel_bc bc_iter > /dev/null 2>&1
python tools/ncu_sass_hot.py gpurun_out/bc_iter.ncu-rep 400 > gpurun_out/bc_iter_hot.txt 2>&1
python tools/ncu_summary.py gpurun_out/bc_iter.ncu-rep > gpurun_out/bc_iter_summary.txt 2>&1
cat gpurun_out/ab_summary.txt; tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bc_iter_summary.txt
