import numpy as np, sys
sys.path.insert(0,'/root/repo')
import paper_2012_14702_b200 as ipt, oracle
R=oracle.ref()
n=130
rng=np.random.default_rng(n)
a=rng.standard_normal((n,n))+1j*rng.standard_normal((n,n))
f=ipt.lu_factor(a)
lu,perm,s=R.lu_factor(a)
d=np.nonzero(f.perm!=perm)[0]
print("first perm diff", d[:5])
print("panel0 L max diff", np.max(np.abs(f.lu[:,:64]-lu[:,:64])))
print("U12 rows 0..63 cols 64.. diff", np.max(np.abs(f.lu[:64,64:]-lu[:64,64:])))
# check trailing after first panel: compute A22 expected = PA[64:,64:] - L21 U12 using our own factors
P=a[f.perm]
L21=f.lu[64:,:64]; U12=f.lu[:64,64:]
# reference unblocked result of column 64 pivot
print("col64 our", f.lu[64:70,64]); print("col64 ref", lu[64:70,64])
