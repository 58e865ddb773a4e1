import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import torch
import test_kernels_gpu as T
for mode in ("flat", "slab"):
    os.environ["RALPB_CONV"] = mode
    for case in [(4, 56, 56, 128, 256, 3, 1), (2, 56, 56, 128, 256, 3, 1), (4, 28, 28, 256, 512, 3, 1), (8, 56, 56, 128, 256, 3, 1), (4, 112, 112, 64, 128, 3, 1)]:
        try:
            T.test_conv_fwd(case); r = "ok"
        except AssertionError as e:
            r = "FAIL " + str(e).splitlines()[2]
        print(mode, case, r, flush=True)
