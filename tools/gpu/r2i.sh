set -x
(for du in 2 4; do timeout 60 ./tools/fz_time 32 65536 65536 1 10 0 $du; done; timeout 60 ./tools/fz_stall 32 65536 65536 1 5 0 2; timeout 60 ./tools/fz_stall 32 65536 65536 1 5 0 4) > gpurun_out/r2i_fz.txt 2>&1
(timeout 60 ./tools/tc_stall 32 65536 65536 1 5) > gpurun_out/r2i_tc_stall.txt 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_solve.py > gpurun_out/r2i_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_memcheck.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_solve.py > gpurun_out/r2i_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_synccheck.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_solve.py > gpurun_out/r2i_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_racecheck.log
