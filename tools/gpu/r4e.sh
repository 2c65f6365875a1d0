for i in 1 2; do timeout 900 python bench.py > gpurun_out/r4e_bench_$i.json 2> gpurun_out/r4e_bench_$i.err; done
