import sys; sys.path.insert(0,'tests')
import numpy as np, paper_2004_02583_b200 as tk
from golden_io import Fixture
ctx = tk.Context(0)
fx = Fixture("t4"); m = fx.meta
eng = tk.FactorEngine.with_als(tk.AlsConfig(eta=m["eta"], seed=m["seed"], max_iters=50))
t, r = ctx.t_hosvd(fx.tensor, tk.Truncation(fx.ranks), eng)
print("single t4", [p.als.iterations for p in r.per_mode], fx.iterations)
# local slab shapes of world 2
a = np.asfortranarray(fx.tensor[..., :3])
for mode in range(1,5):
    l = np.random.default_rng(mode).standard_normal((a.shape[mode-1], 3))
    x = ctx.unfold_t_times(a, mode, l)
    mm = np.random.default_rng(mode).standard_normal((a.size//a.shape[mode-1], 3))
    y = ctx.unfold_times(a, mode, mm)
print("prims ok")
b = np.asfortranarray(fx.tensor[:, :, :4, :])
for mode in range(1,5):
    mm = np.random.default_rng(mode).standard_normal((b.size//b.shape[mode-1], 2))
    y = ctx.unfold_times(b, mode, mm)
    l = np.random.default_rng(mode).standard_normal((b.shape[mode-1], 2))
    x = ctx.unfold_t_times(b, mode, l)
print("prims2 ok")
