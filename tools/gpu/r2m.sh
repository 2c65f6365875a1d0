for i in 1 2 3; do
timeout 60 ./tools/fz_stall_prev 32 65536 65536 1 5 0 | grep -E "ms per launch|latency|per row" | sed 's/^/prev /'
timeout 60 ./tools/fz_stall 32 65536 65536 1 5 0 | grep -E "ms per launch|latency|per row" | sed 's/^/new  /'
done > gpurun_out/r2m_ab.txt 2>&1
