OOCNMF_PROFILE_IO=1 timeout 900 python bench.py > gpurun_out/r3h_bench.json 2> gpurun_out/r3h_bench.err
