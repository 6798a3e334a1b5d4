"""ncu target: a few complete m-Cubes runs (run path: vsample -> reduce -> finish with grid refinement)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_05730_b200 as pb
fam, d, n = sys.argv[1], int(sys.argv[2]), int(float(sys.argv[3]))
for _ in range(3):
    r = pb.mcubes_run(pb.get_integrand(fam, d), n, d, 4, seed=0)
print(r.estimate, r.errorest)
