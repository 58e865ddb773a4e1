"""RALP_MPS (sharded FC tail) at W=1 against numpy: logits of one step from the FC-0 output and
the bf16-rounded FC-1 weights (usage: tools/check_mps_w1.py [single|multi])."""
import sys, ctypes as C
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_1901_05803_b200 import synthetic, _lib
from paper_1901_05803_b200.executor import RankExecutor, lower
from paper_1901_05803_b200.planner import JobSpec, Strategy, catalog_lookup

mode = sys.argv[1] if len(sys.argv) > 1 else "multi"
model = catalog_lookup("cifar_small").with_batch_size(32)
ex = RankExecutor(JobSpec(model, Strategy.ralp(4), 1), fc_sharding=mode)
params = synthetic.init_params(ex.layers, 1)
ex.set_params(params)
imgs, labs = synthetic.batch(1, 0, 0, 32, ex.in_shape, ex.classes)
ex.step(imgs, labs)
st = ex.stats()
def rd(which, dt):
    n = _lib.lib().ralpb_model_debug_buffer(ex._h, 0, which, None)
    b = np.zeros(n, dtype=dt)
    _lib.lib().ralpb_model_debug_buffer(ex._h, 0, which, b.ctypes.data_as(C.c_void_p))
    return b
lg = rd(2, np.float32).reshape(32, -1)[:, :10]
h = rd(3, np.uint16)
h0 = (h.astype(np.uint32) << 16).view(np.float32).reshape(32, -1)
w1, b1 = params[5]
w1u = w1.astype(np.float32).view(np.uint32)
w1b = (((w1u + 0x7FFF + ((w1u >> 16) & 1)) >> 16) << 16).astype(np.uint32).view(np.float32)
ref = h0 @ w1b.T + b1
print(mode, "loss", st.loss, "logits err", float(np.abs(lg - ref).max()), "row0", lg[0, :4], "ref", ref[0, :4])
