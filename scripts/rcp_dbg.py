import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2302_05730_b200 import _native
rng = np.random.default_rng(11)
sets = {
 "unit": rng.random(2_000_000) + 1e-4,
 "a2range": 0.0004 + 0.25 * rng.random(1_000_000),
 "anyexp": np.ldexp(1.0 + rng.random(1_000_000), rng.integers(-900, 900, 1_000_000)),
 "below_pow2": np.nextafter(np.ldexp(1.0, np.arange(-100, 100)), 0),
 "above_pow2": np.nextafter(np.ldexp(1.0, np.arange(-100, 100)), 4),
 "pow2": np.ldexp(1.0, np.arange(-100, 100)),
 "one_plus": 1.0 + np.ldexp(1.0, -np.arange(1, 53)),
 "two_minus": 2.0 - np.ldexp(1.0, -np.arange(1, 53)),
 "neg": -(rng.random(1000) + 0.5),
}
for k, x in sets.items():
    got = _native.debug_divide(x, 0); want = 1.0 / x
    bad = np.nonzero(got != want)[0]
    print(k, x.size, "mismatches", bad.size, [(x[i].hex(), got[i].hex(), want[i].hex()) for i in bad[:3]])
