# GPU session 6: ResNet-50 tests (teacher-forced blocks), bench N=1 with all comparators
set -x
timeout 1500 python -m pytest tests/test_resnet_gpu.py -q -s > gpurun_out/t_resnet.log 2>&1; echo resnet rc $?
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench6.log 2>&1; echo bench rc $?
tail -n 3 gpurun_out/t_resnet.log
