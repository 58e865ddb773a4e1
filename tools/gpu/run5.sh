# GPU session 5: ResNet-50 executed, step tests (conv back segment), fp32 parity, the dominant kernel's ncu capture
set -x
timeout 1500 python -m pytest tests/test_resnet_gpu.py -q -s -x > gpurun_out/t_resnet.log 2>&1; echo resnet rc $?
timeout 1500 python -m pytest tests/test_step_gpu.py tests/test_parity_fp32_gpu.py -q -s > gpurun_out/t_step.log 2>&1; echo step rc $?
python tools/step_launches.py 1 > gpurun_out/plain_steps.log 2>&1 && echo plain ok
for spec in "conv_slab_fwd_kernel<.int.3, .int.4, .int.1, .bool.1>:2" "conv_slab_fwd_kernel<.int.3, .int.4, .int.1, .bool.0>:0" "conv_slab_fwd_kernel<.int.3, .int.4, .int.2, .bool.1>:1"; do
  pat="${spec%:*}"; skip="${spec##*:}"
  tag=$(echo "$pat" | tr -c 'a-z0-9_' '_' | cut -c1-48)
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$pat" -s $skip -c 1 -o gpurun_out/prof_$tag python tools/step_launches.py 1 > gpurun_out/ncu_$tag.log 2>&1; echo cap $tag rc $?
done
tail -n 3 gpurun_out/t_resnet.log gpurun_out/t_step.log
