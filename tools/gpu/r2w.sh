# 4-GPU box: multi-GPU / distributed tests (incl. the dead-rank test and the opt-in variants), scaling lines
set -x
nvidia-smi topo -m > gpurun_out/r2w_topo.txt 2>&1
timeout 1500 python -m pytest tests/test_multi_gpu.py tests/test_gpu_distributed.py -q -rf -p no:cacheprovider > gpurun_out/r2w_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2w_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e-f64 > gpurun_out/r2w_bench_n1.json 2> gpurun_out/r2w_bench_n1.err
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2970$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/r2w_bench_n$n.json 2> gpurun_out/r2w_bench_n$n.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29711 bench.py --gpus 4 --steps 20 --warmup 5 --scaling weak --no-e2e > gpurun_out/r2w_bench_weak4.json 2> gpurun_out/r2w_bench_weak4.err
