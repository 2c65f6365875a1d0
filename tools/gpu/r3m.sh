# 4 GPUs: out-of-core at N=4 (concurrent host links), N=1 on the same box for the ratio
set -x
free -g > gpurun_out/r3m_mem.txt; nproc >> gpurun_out/r3m_mem.txt
timeout 900 python bench.py --workload ooc --ooc-gb 16 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r3m_ooc_n1.json 2> gpurun_out/r3m_ooc_n1.err
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29671 bench.py --gpus 4 --workload ooc --ooc-gb 16 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r3m_ooc_n4.json 2> gpurun_out/r3m_ooc_n4.err
