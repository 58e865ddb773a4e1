# GPU session 15: fused BN statistics (GEMM colstats) + warp-per-row im2col: resnet / branchy tests,
# launch lists, bench
set -x
timeout 900 python -m pytest tests/test_resnet_gpu.py tests/test_branchy_gpu.py -q -s > gpurun_out/t_rb15.log 2>&1; echo tests rc $?
timeout 600 python tools/model_launches.py inception-v3 4 > gpurun_out/inc_plain15.log 2>&1; echo plain rc $?
timeout 600 python tools/model_launches.py resnet-50 4 > gpurun_out/res_plain15.log 2>&1; echo plain rc $?
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_inception15.csv python tools/model_launches.py inception-v3 2 > gpurun_out/ncu_inc15.log 2>&1; echo list rc $?
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_resnet15.csv python tools/model_launches.py resnet-50 2 > gpurun_out/ncu_res15.log 2>&1; echo list rc $?
timeout 900 python bench.py --steps 10 --warmup 3 --no-fp32 > gpurun_out/bench15.json 2> gpurun_out/bench15.err; echo bench rc $?
tail -3 gpurun_out/t_rb15.log; tail -1 gpurun_out/inc_plain15.log; tail -1 gpurun_out/res_plain15.log
