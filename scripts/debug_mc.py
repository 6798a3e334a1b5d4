import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PCB_MCUBES_SEGMENTS"]="1"
import numpy as np
import paper_2302_05730_b200 as pb
from paper_2302_05730_b200 import _native, vegas
from oracle import parcube_oracle as po
fam,d,n="f2",6,300000
plan, oplan = pb.make_plan(n, d), po.make_plan(n, d)
t = vegas.BinContributions(d, 500); t.c[:] = np.linspace(0.0, 1.0, 500) ** 6
grid = pb.refine_grid(pb.init_grid(d), t)
it, c, gp = _native.mcubes_sample(pb.get_integrand(fam,d).device_spec(), plan, grid.boundaries, 77, want_group_partials=True)
want = po.vsample(fam, oplan, grid.boundaries, seed=77, workers=4)
wgp = want["group_partials"]
bad = np.nonzero((gp[:,0]!=wgp[:,0])|(gp[:,1]!=wgp[:,1]))[0]
print("groups differing", bad[:20], len(bad), "of", len(gp))
for gidx in bad[:3]:
    print(gidx, gp[gidx], wgp[gidx])
# uniform grid too
grid0 = pb.init_grid(d)
it, c, gp = _native.mcubes_sample(pb.get_integrand(fam,d).device_spec(), plan, grid0.boundaries, 77, want_group_partials=True)
want = po.vsample(fam, oplan, grid0.boundaries, seed=77, workers=4)
print("uniform grid groups differing", np.count_nonzero(gp!=want["group_partials"]))
# which boundaries trigger? check transform on random y
y = np.random.default_rng(0).random((200000, d))
gx, gj, gb = vegas.transform_many(y, grid)
ox, oj, ob = po.grid_transform(y, grid.boundaries)
print("transform equal", np.array_equal(gx,ox), np.array_equal(gj,oj), np.array_equal(gb,ob))
