(for r in 65536 16384 8192; do timeout 60 ./tools/fu_bench 32 $r 1; done; timeout 60 ./tools/fu_bench_prof 32 65536 1) > gpurun_out/r3y_fu.txt 2>&1
