# GPU session 19: two epilogue warpgroups in the GEMM engine -- full single-GPU suite, ResNet / Inception
# step times, quick headline bench, ResNet launch list
set -x
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/t_full19.log 2>&1; echo tests rc $?
timeout 600 python tools/model_launches.py resnet-50 4 > gpurun_out/res_plain19.log 2>&1; echo plain rc $?
timeout 600 python tools/model_launches.py inception-v3 4 > gpurun_out/inc_plain19.log 2>&1; echo plain rc $?
timeout 600 python bench.py --steps 20 --warmup 5 --quick > gpurun_out/bench19.json 2> gpurun_out/bench19.err; echo bench rc $?
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_resnet19.csv python tools/model_launches.py resnet-50 2 > gpurun_out/ncu_res19.log 2>&1; echo list rc $?
tail -3 gpurun_out/t_full19.log; tail -1 gpurun_out/res_plain19.log; tail -1 gpurun_out/inc_plain19.log; cut -c1-300 gpurun_out/bench19.json
