set -x
timeout 1500 python -m pytest tests/test_branchy_gpu.py -q -x > gpurun_out/t_42.log 2>&1; echo tests rc $?
for i in 1 2; do for mdl in inception-v3 googlenet; do timeout 300 python tools/model_launches.py $mdl 6 2>/dev/null; done; done
tail -2 gpurun_out/t_42.log
