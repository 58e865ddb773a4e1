# GPU session 18 (4 GPUs): quick bench (bucketed vs unbucketed sync) + multi-rank parity at W=4
set -x
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29672 bench.py --gpus $N --steps 20 --warmup 5 --quick > gpurun_out/mg_bench18_n$N.log 2>&1; echo bench rc $?
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29671 tests/multi_rank_parity.py > gpurun_out/mg_parity18_n$N.log 2>&1; echo parity rc $?
tail -n 2 gpurun_out/mg_parity18_n$N.log
