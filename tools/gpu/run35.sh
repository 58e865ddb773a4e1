# GPU session 35: residual-add GEMM epilogue (shortcut / branch gradients summed in the dgrad GEMM)
set -x
timeout 2400 python -m pytest tests/test_resnet_gpu.py tests/test_branchy_gpu.py tests/test_step_gpu.py tests/test_headline_parity_gpu.py tests/test_kernels_gpu.py -q -x > gpurun_out/t_35.log 2>&1; echo tests rc $?
timeout 600 python tools/model_launches.py resnet-50 4 > gpurun_out/res_plain35.log 2>&1; echo plain rc $?
timeout 600 python tools/model_launches.py inception-v3 4 > gpurun_out/inc_plain35.log 2>&1; echo plain rc $?
timeout 600 python tools/model_launches.py googlenet 4 > gpurun_out/goo_plain35.log 2>&1; echo plain rc $?
tail -2 gpurun_out/t_35.log; tail -1 gpurun_out/res_plain35.log; tail -1 gpurun_out/inc_plain35.log; tail -1 gpurun_out/goo_plain35.log
