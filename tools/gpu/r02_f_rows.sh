# Round-2 re-measurement of the F1 (multi-tenant) and BASELINE cfg 4 (streamed 10M-trial YET) lines
# with the current kernels, one GPU.
mkdir -p gpurun_out
timeout 900 python tools/multitenant.py > gpurun_out/r02_mt_p1.json 2> gpurun_out/r02_mt_p1.err
timeout 1200 python tools/stream_bench.py > gpurun_out/r02_stream10m_n1.json 2> gpurun_out/r02_stream10m_n1.err
cut -c1-1500 gpurun_out/r02_mt_p1.json; echo; cut -c1-1500 gpurun_out/r02_stream10m_n1.json; tail -3 gpurun_out/r02_mt_p1.err gpurun_out/r02_stream10m_n1.err
