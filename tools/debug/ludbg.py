import sys
import numpy as np
sys.path.insert(0, '/root/repo')
import paper_2012_14702_b200 as ipt, oracle
R = oracle.ref()
for n in [int(x) for x in sys.argv[1:]] or [130]:
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    f = ipt.lu_factor(a)
    lu, perm, s = R.lu_factor(a)
    d = np.nonzero(f.perm != perm)[0]
    print(n, "first perm diff", d[:5], "max |lu diff| first 64 rows", np.max(np.abs(f.lu[:64] - lu[:64])),
          "all", np.max(np.abs(f.lu - lu)), flush=True)
