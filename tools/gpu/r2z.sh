set -x
PYTHONPATH=. timeout 900 python tools/fused_crossover.py --d=1,2,3,4,6 --k=16,32 16384x8192 32768x16384 65536x16384 32768x32768 65536x32768 > gpurun_out/r2z_lag.jsonl 2> gpurun_out/r2z_lag.err
