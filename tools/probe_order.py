"""Is the e2e > value gap in bench.py an ordering (clock/power) effect?  Times the
device-resident run, the host-input e2e run and the device-resident run again, twice."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
import bench  # noqa: E402

ex, job, rep = bench._build_executor("ralp", 1, 0)
g = torch.Generator(device="cuda").manual_seed(1234)
shape = ex.in_shape
dimgs = [torch.randn(bench.BATCH, *shape, generator=g, device="cuda") for _ in range(2)]
dlabs = [torch.randint(0, ex.classes, (bench.BATCH,), generator=g, device="cuda", dtype=torch.int32) for _ in range(2)]
himgs = [x.cpu().pin_memory() for x in dimgs]
hlabs = [x.cpu().pin_memory() for x in dlabs]
for r in range(3):
    for name, (i, l, oh, rl) in {"device": (dimgs, dlabs, False, False), "e2e": (himgs, hlabs, True, True),
                                 "device_rl": (dimgs, dlabs, False, True)}.items():
        ms = bench._time_steps(ex, i, l, 20, 5, 1, on_host=oh, read_loss=rl)
        print(f"round {r} {name:10s} {ms:.3f} ms/step  {bench.BATCH / ms * 1e3:.0f} img/s", flush=True)
