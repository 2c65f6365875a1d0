for i in 1 2; do
for v in 1 0; do
OOCNMF_SHARD_H=$v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 90)) bench.py --gpus 2 --workload sparse --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r4y_s$v.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/r4y_s$v.json'));print('N=2 shard_h=$v', round(d['value'],1), {k:round(v,3) for k,v in d['phase_ms_per_step'].items()})" >> gpurun_out/r4y_summary.txt
done; done
