# GPU session 16 (2 GPUs): multi-rank parity incl. whole-layer PS shards and GoogLeNet modules, N=2 bench,
# then single-GPU launch lists for ResNet-50 / Inception-v3 (BN statistics pass restored, warp im2col)
set -x
N=$(nvidia-smi -L | wc -l)
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29651 tests/multi_rank_parity.py > gpurun_out/mg_parity16_n$N.log 2>&1; echo parity rc $?
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29652 bench.py --gpus $N --steps 10 --warmup 3 --no-fp32 > gpurun_out/mg_bench16_n$N.log 2>&1; echo bench rc $?
timeout 600 python tools/model_launches.py inception-v3 4 > gpurun_out/inc_plain16.log 2>&1; echo plain rc $?
timeout 600 python tools/model_launches.py resnet-50 4 > gpurun_out/res_plain16.log 2>&1; echo plain rc $?
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_inception16.csv python tools/model_launches.py inception-v3 2 > gpurun_out/ncu_inc16.log 2>&1; echo list rc $?
tail -n 3 gpurun_out/mg_parity16_n$N.log; tail -1 gpurun_out/inc_plain16.log; tail -1 gpurun_out/res_plain16.log
