"""Dev: device slab operators vs the oracle local operator, one process."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1])); sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np, torch
import oracle as O
from paper_2012_06646_b200 import ib, slab as S
import test_slab as T
print("start", flush=True)
ext, h, alpha, per, n = (32, 24, 40), 0.5, (0.5, 0.5, 0.0), (True, True, True), 6000
rng = np.random.default_rng(5)
pts = np.stack([rng.uniform(0, ext[a] * h, n) for a in range(3)], axis=1)
vals = rng.uniform(-1, 1, n)
grid = ib.StaggeredGrid(list(ext), h, list(alpha), list(per))
og = O.make_grid(list(ext), h, list(alpha), list(per))
X = torch.tensor(pts, device="cuda")
planes = S.home_planes(grid, X); torch.cuda.synchronize(); print("planes ok", flush=True)
print(np.array_equal(planes.cpu().numpy(), O.home_cells(og, pts)[:, -1]), flush=True)
for world in (1, 2):
    for rank in range(world):
        dec = S.SlabDecomposition(grid, rank, world)
        sp, ip = T._oracle_local_ops(dec, ext, h, alpha, per)
        mine = (S.owner_of_planes(planes, ext[-1], world) == rank)
        Xm = X[mine].contiguous(); Gm = torch.tensor(vals, device="cuda")[mine].contiguous()
        print("world", world, "rank", rank, "n", int(mine.sum()), dec.lay, flush=True)
        got = dec._spread(Xm, Gm); torch.cuda.synchronize(); print("spread ok", flush=True)
        want = sp(Xm.cpu(), Gm.cpu())
        print("local spread dev", O.max_rel_deviation(got.cpu().numpy(), want.numpy()), flush=True)
        F = torch.rand(dec.local.point_count(), dtype=torch.float64, device="cuda")
        e = dec._interp(F, Xm); torch.cuda.synchronize()
        print("local interp dev", O.max_rel_deviation(e.cpu().numpy(), ip(F.cpu(), Xm.cpu()).numpy()), flush=True)
