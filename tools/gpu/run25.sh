set -x
N=$(nvidia-smi -L | wc -l)
RALPB_PARITY_ONLY=resnet-50 timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29691 tests/multi_rank_parity.py > gpurun_out/mg_parity25_n$N.log 2>&1; echo parity rc $?
tail -n 30 gpurun_out/mg_parity25_n$N.log | cut -c1-200
