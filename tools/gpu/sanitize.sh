mkdir -p gpurun_out
timeout 300 python tests/gpu_sanitize_tiny.py > gpurun_out/san_plain.log 2>&1 && \
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python tests/gpu_sanitize_tiny.py > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san_memcheck.log
tail -5 gpurun_out/san_plain.log; tail -8 gpurun_out/san_memcheck.log
