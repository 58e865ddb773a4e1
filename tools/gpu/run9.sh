set -x
timeout 900 python -m pytest tests/test_resnet_gpu.py -q -s > gpurun_out/t_resnet9.log 2>&1; echo resnet rc $?
tail -5 gpurun_out/t_resnet9.log
