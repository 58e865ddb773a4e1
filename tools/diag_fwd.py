"""Run the forward-conv kernel test at extra VGG shapes under both kernel families
(RALPB_CONV=flat|slab) and print ok/FAIL per case (debug aid; needs a GPU)."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import test_kernels_gpu as T  # noqa: E402

CASES = [(4, 56, 56, 128, 256, 3, 1), (2, 56, 56, 128, 256, 3, 1), (4, 28, 28, 256, 512, 3, 1),
         (8, 56, 56, 128, 256, 3, 1), (4, 112, 112, 64, 128, 3, 1), (2, 224, 224, 64, 64, 3, 1)]
for mode in ("flat", "slab"):
    os.environ["RALPB_CONV"] = mode
    for case in CASES:
        try:
            T.test_conv_fwd(case)
            r = "ok"
        except AssertionError as e:
            r = "FAIL " + str(e).splitlines()[2]
        print(mode, case, r, flush=True)
