(for m in 8192 16384 32768 65536; do
  timeout 60 ./tools/fz_time 32 $m 65536 1 10 0 | grep "ms per"
  timeout 60 ./tools/tc_stall 32 $m 65536 1 10 | grep "ms per"
done) > gpurun_out/r2v_shapes.txt 2>&1
for m in 8192 16384; do
timeout 300 python bench.py --m $m --steps 30 --warmup 5 --no-sparse --no-e2e --no-cpu-baseline > gpurun_out/r2v_bench_m$m.json 2>/dev/null
OOCNMF_FUSED=0 timeout 300 python bench.py --m $m --steps 30 --warmup 5 --no-sparse --no-e2e --no-cpu-baseline > gpurun_out/r2v_bench_m${m}_2p.json 2>/dev/null
done
