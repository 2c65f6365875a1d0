# 4-GPU box: distributed tests, sparse all-gather overlap and dense sharded-H A/B
set -x
timeout 1200 python -m pytest tests/test_multi_gpu.py tests/test_gpu_distributed.py -q -rf -p no:cacheprovider > gpurun_out/r2o_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2o_pytest.log
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $1 bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline "${@:3}" > gpurun_out/r2o_$2.json 2> gpurun_out/r2o_$2.err; }
run 29601 sparse_ov --workload sparse
OOCNMF_AG_OVERLAP=0 run 29602 sparse_noov --workload sparse
run 29603 dense_shard --no-sparse
OOCNMF_SHARD_H=0 run 29604 dense_noshard --no-sparse
