timeout 60 ./tools/fz_stall 32 65536 65536 1 5 0 > gpurun_out/r2n_fz.txt 2>&1
timeout 60 ./tools/fz_stall 32 65536 65536 1 5 0 >> gpurun_out/r2n_fz.txt 2>&1
