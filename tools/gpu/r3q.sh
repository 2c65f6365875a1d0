set -x
timeout 1200 python -m pytest tests/test_multi_gpu.py -q -rf -p no:cacheprovider -k "nvls or csr_sharded or csr_rnmf" > gpurun_out/r3q_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r3q_pytest.log
for i in 1 2; do
OOCNMF_NVLS=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2969$i bench.py --gpus 4 --workload sparse --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r3q_sparse_nvls4_$i.json 2> gpurun_out/r3q_sparse_nvls4_$i.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2968$i bench.py --gpus 4 --workload sparse --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r3q_sparse_base4_$i.json 2> gpurun_out/r3q_sparse_base4_$i.err
done
