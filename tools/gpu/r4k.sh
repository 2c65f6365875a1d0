set -x
timeout 1800 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/r4k_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r4k_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4k_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/r4k_smoke.log
timeout 900 python bench.py > gpurun_out/r4k_bench_n1.json 2> gpurun_out/r4k_bench_n1.err
for n in 2 4; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2977$n bench.py --gpus $n > gpurun_out/r4k_bench_n$n.json 2> gpurun_out/r4k_bench_n$n.err
done
