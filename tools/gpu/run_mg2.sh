# Multi-GPU session 2: the full GPU suite on a 2-GPU box (incl. the multi-rank parity scripts) and the bench at N=2
set -x
N=$(nvidia-smi -L | wc -l)
timeout 2400 python -m pytest tests -m gpu -q -k "not headline and not resnet and not fp32" > gpurun_out/mg_tests_n$N.log 2>&1; echo tests rc $?
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29641 tests/multi_rank_parity.py > gpurun_out/mg_parity_n$N.log 2>&1; echo parity rc $?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29642 bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/mg_bench_n$N.log 2>&1; echo bench rc $?
tail -n 5 gpurun_out/mg_tests_n$N.log gpurun_out/mg_parity_n$N.log
