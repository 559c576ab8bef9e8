cd $GRAFT_REPO_ROOT
for rf in 0 1; do
DGAS_ND_REFINE=$rf timeout 900 python - <<'PY' >> gpurun_out/cfg3_refine.log 2>&1
import os, numpy as np, torch, dgas_gen as g
from paper_1903_11357_b200 import dgas
P = g.config(3); S = dgas.Solver(P)
r = g.normal(42, S.N)
z = S.apply(torch.from_numpy(r).cuda()).cpu().numpy()
zr = np.load('tools/cfg3_z_refined.npy')
sample=[0, P.n_sub//3, P.n_sub-1]
mask=np.zeros(P.n_cells,bool)
for s in sample: mask|=P.part==s
idx=np.repeat(mask, S.info['n_p'])
print('refine', os.environ['DGAS_ND_REFINE'], 'sampled rel err vs refined oracle', np.linalg.norm(z[idx]-zr[idx])/np.linalg.norm(zr[idx]))
PY
done
cat gpurun_out/cfg3_refine.log
