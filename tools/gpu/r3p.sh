set -x
timeout 1200 python -m pytest tests/test_multi_gpu.py -q -rf -p no:cacheprovider -k "nvls or csr_sharded or csr_rnmf" > gpurun_out/r3p_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r3p_pytest.log
OOCNMF_NVLS=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29681 bench.py --gpus 2 --workload sparse --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r3p_sparse_nvls2.json 2> gpurun_out/r3p_sparse_nvls2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29682 bench.py --gpus 2 --workload sparse --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r3p_sparse_base2.json 2> gpurun_out/r3p_sparse_base2.err
