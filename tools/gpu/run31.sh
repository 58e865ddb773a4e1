# GPU session 31: shared-memory staged first-layer im2col + 32-bit pool kernels
set -x
timeout 2400 python -m pytest tests/test_kernels_gpu.py tests/test_step_gpu.py tests/test_resnet_gpu.py tests/test_branchy_gpu.py tests/test_parity_fp32_gpu.py -q -x > gpurun_out/t_31.log 2>&1; echo tests rc $?
timeout 600 python tools/model_launches.py alexnet 4 > gpurun_out/alex_plain31.log 2>&1; echo plain rc $?
timeout 600 python tools/model_launches.py resnet-50 4 > gpurun_out/res_plain31.log 2>&1; echo plain rc $?
timeout 600 python tools/model_launches.py googlenet 4 > gpurun_out/goo_plain31.log 2>&1; echo plain rc $?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_alexnet31.csv python tools/model_launches.py alexnet 2 > gpurun_out/ncu_alex31.log 2>&1; echo list rc $?
tail -2 gpurun_out/t_31.log; tail -1 gpurun_out/alex_plain31.log; tail -1 gpurun_out/res_plain31.log; tail -1 gpurun_out/goo_plain31.log
