set -x
for cfg in c2 c3 c5; do for sh in rows columns; do
TMB_BENCH_SMOKE_1GPU=1 timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config $cfg --steps 2 --warmup 3 --shard $sh 2>gpurun_out/r02q_smk_${cfg}_${sh}.err | tail -1 | cut -c1-400
done; done
