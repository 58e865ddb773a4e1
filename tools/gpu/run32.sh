# GPU session 32: im2col lane-tap indexing; ncu of the AlexNet first-layer im2col and pool-backward gather
set -x
timeout 1200 python -m pytest tests/test_kernels_gpu.py tests/test_resnet_gpu.py -q -x -k "im2col or first or resnet50_fc or teacher" > gpurun_out/t_32.log 2>&1; echo tests rc $?
timeout 600 python tools/model_launches.py alexnet 4 > gpurun_out/alex_plain32.log 2>&1; echo plain rc $?
timeout 600 python tools/model_launches.py resnet-50 4 > gpurun_out/res_plain32.log 2>&1; echo plain rc $?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"pack_im2col_smem|maxpool_bwd_gather" -c 3 -o gpurun_out/prof_alex_im2col_pool python tools/model_launches.py alexnet 1 > gpurun_out/ncu_alex32.log 2>&1; echo ncu rc $?
tail -2 gpurun_out/t_32.log; tail -1 gpurun_out/alex_plain32.log; tail -1 gpurun_out/res_plain32.log
