import numpy as np, sys
sys.path.insert(0,'.')
from paper_2408_12479_b200 import emfgpu as G
g=np.load('tests/golden/stability.npz')
e,i=G.stability_sweep(g['scales'],200,42)
print("invalid equal:", np.array_equal(i,g['inv']), np.abs(i-g['inv']).sum())
ref=g['err']
eq = e==ref
print("bitwise equal cells:", eq.sum(), "of", eq.size)
rel = np.abs(e-ref)/np.maximum(ref,1e-300)
names=[f"{m}/{f}/{q}" for m in G.SWEEP_MODELS for f in G.SWEEP_FORMULATIONS for q in G.SWEEP_QUANTITIES]
for c in range(32):
    bad = ~eq[:,c]
    if bad.any(): print(names[c], bad.sum(), "max rel diff %.3e"%rel[:,c].max(), "scales", np.round(np.log10(g['scales'][bad]),1)[:8])
