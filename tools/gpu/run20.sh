# GPU session 20: wave-aware GEMM tile width -- ResNet / Inception / GoogLeNet step times, quick headline bench, tests
set -x
timeout 600 python tools/model_launches.py resnet-50 4 > gpurun_out/res_plain20.log 2>&1; echo plain rc $?
timeout 600 python tools/model_launches.py inception-v3 4 > gpurun_out/inc_plain20.log 2>&1; echo plain rc $?
timeout 600 python tools/model_launches.py googlenet 4 > gpurun_out/goo_plain20.log 2>&1; echo plain rc $?
timeout 600 python bench.py --steps 20 --warmup 5 --quick > gpurun_out/bench20.json 2> gpurun_out/bench20.err; echo bench rc $?
timeout 1800 python -m pytest tests/test_resnet_gpu.py tests/test_branchy_gpu.py tests/test_headline_parity_gpu.py tests/test_step_gpu.py -q -x > gpurun_out/t_20.log 2>&1; echo tests rc $?
tail -1 gpurun_out/res_plain20.log; tail -1 gpurun_out/inc_plain20.log; tail -1 gpurun_out/goo_plain20.log; cut -c1-200 gpurun_out/bench20.json; tail -2 gpurun_out/t_20.log
