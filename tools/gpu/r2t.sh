for i in 1 2; do
timeout 60 ./tools/fz_stall 32 65536 65536 1 5 0 | grep -E "ms per launch|latency|per row|offset" | sed 's/^/plan0 /'
OOCNMF_FUSED_PLAN=1 timeout 60 ./tools/fz_stall 32 65536 65536 1 5 0 | grep -E "ms per launch|latency|per row|offset" | sed 's/^/plan1 /'
done > gpurun_out/r2t_ab.txt 2>&1
