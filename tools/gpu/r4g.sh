for i in 1 2; do OOCNMF_PROFILE_IO=1 timeout 900 python bench.py --no-sparse --no-cpu-baseline > gpurun_out/r4g_bench_$i.json 2> gpurun_out/r4g_bench_$i.err; done
