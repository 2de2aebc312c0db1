"""Which intermediate of a deterministic-mode step differs between two runs."""
import sys
import torch
sys.path.insert(0, "tests")
sys.path.insert(0, ".")
from conftest import load_golden, golden_scene  # noqa: E402
import test_gpu_deterministic as T  # noqa: E402
from paper_2503_23044_b200.trainer import TrainConfig, TrainState, train_step  # noqa: E402

d = load_golden("train_small")
views, images, priors, npri = T._inputs(d)
runs = []
for _ in range(2):
    st = TrainState(golden_scene(d), TrainConfig(**T._cfg(True)))
    keep = []
    train_step(st, views, images, priors, normal_priors=npri, keep=keep)
    torch.cuda.synchronize()
    runs.append((st, keep))
(a, ka), (b, kb) = runs
for vi, (x, y) in enumerate(zip(ka, kb)):
    print(vi, "grad_splat", torch.equal(x.grad_splat, y.grad_splat))
    for k in x.grad_gauss:
        print(vi, "gg", k, torch.equal(x.grad_gauss[k], y.grad_gauss[k]))
    print(vi, "R.rgb", torch.equal(x.raster.rgb, y.raster.rgb), "tlist",
          torch.equal(x.bins.tile_list, y.bins.tile_list))
for name in a.flat.layout:
    try:
        ga, gb = a.flat.view(a.flat.grad, name), b.flat.view(b.flat.grad, name)
        print("grad", name, torch.equal(ga, gb), float((ga - gb).abs().max()))
    except Exception as e:  # noqa: BLE001
        print(name, e)
print("flat grad equal", torch.equal(a.flat.grad, b.flat.grad))
diff = (a.flat.grad - b.flat.grad).abs()
idx = torch.nonzero(diff).flatten()
print("n diff", idx.numel(), idx[:20].tolist())
print("layout", {k: v for k, v in list(a.flat.layout.items())[:20]})
