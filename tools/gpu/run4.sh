# GPU session 4: fp32 parity (thresholds + teacher-forced layers), step tests incl. the conv back segment
set -x
timeout 1500 python -m pytest tests/test_parity_fp32_gpu.py -q -s > gpurun_out/t_fp32.log 2>&1; echo fp32 rc $?
timeout 1500 python -m pytest tests/test_step_gpu.py -q -s > gpurun_out/t_step.log 2>&1; echo step rc $?
timeout 1500 python -m pytest tests -m gpu -q -x -k "not fp32 and not step_gpu and not headline" > gpurun_out/t_rest.log 2>&1; echo rest rc $?
tail -n 3 gpurun_out/t_fp32.log gpurun_out/t_step.log gpurun_out/t_rest.log
