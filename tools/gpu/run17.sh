# GPU session 17 (2 GPUs): bucketed parameter sync under the backward -- multi-rank parity + quick bench
set -x
N=$(nvidia-smi -L | wc -l)
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29661 tests/multi_rank_parity.py > gpurun_out/mg_parity17_n$N.log 2>&1; echo parity rc $?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29662 bench.py --gpus $N --steps 20 --warmup 5 --quick > gpurun_out/mg_bench17_n$N.log 2>&1; echo bench rc $?
tail -n 2 gpurun_out/mg_parity17_n$N.log; grep -h '^{' gpurun_out/mg_bench17_n$N.log | tail -1 | cut -c1-600
