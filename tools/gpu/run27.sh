set -x
N=$(nvidia-smi -L | wc -l)
RALPB_PARITY_ONLY=resnet-50 timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29701 tests/multi_rank_parity.py > gpurun_out/mg_parity27a_n$N.log 2>&1; echo parity rc $?
RALPB_PARITY_ONLY=inception-v3 timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29702 tests/multi_rank_parity.py > gpurun_out/mg_parity27b_n$N.log 2>&1; echo parity rc $?
grep -E "step|PARITY|!=|differ" gpurun_out/mg_parity27a_n$N.log gpurun_out/mg_parity27b_n$N.log | cut -c1-200
