# 4 GPUs: distributed / CLI tests, dense N=2/4 bench, sparse N=4 with the replicated H update
set -x
timeout 1500 python -m pytest tests/test_multi_gpu.py tests/test_gpu_distributed.py tests/test_cli_gpu.py -q -rf -p no:cacheprovider > gpurun_out/r3j_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r3j_pytest.log
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/r3j_bench_n$n.json 2> gpurun_out/r3j_bench_n$n.err
done
OOCNMF_SHARD_H=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29655 bench.py --gpus 4 --workload sparse --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r3j_sparse_rep4.json 2> gpurun_out/r3j_sparse_rep4.err
