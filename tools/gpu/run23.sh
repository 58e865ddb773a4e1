set -x
timeout 1200 python -m pytest tests/test_resnet_gpu.py tests/test_branchy_gpu.py -q -x > gpurun_out/t_23.log 2>&1; echo tests rc $?
timeout 600 python tools/model_launches.py resnet-50 4 > gpurun_out/res_plain23.log 2>&1; echo plain rc $?
timeout 600 python tools/model_launches.py inception-v3 4 > gpurun_out/inc_plain23.log 2>&1; echo plain rc $?
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_resnet23.csv python tools/model_launches.py resnet-50 2 > gpurun_out/ncu_res23.log 2>&1; echo list rc $?
tail -2 gpurun_out/t_23.log; tail -1 gpurun_out/res_plain23.log; tail -1 gpurun_out/inc_plain23.log
