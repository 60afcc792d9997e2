mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_random_gpu.py -q -p no:cacheprovider > gpurun_out/pytest_rand.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_rand.log
tail -15 gpurun_out/pytest_rand.log
