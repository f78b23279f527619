import sys; sys.path.insert(0,'/root/repo')
import numpy as np, torch, oracle
from paper_2406_05128_b200 import params
d=np.load('/root/repo/tests/golden/golden_framewise.npz')
i=3; k=f"f{i}_"
T1,hop,M=(int(x) for x in d[k+"cfg"])
e,fr,g=d[k+"e"],d[k+"frames"],d[k+"g"]
plan=params.FramePlan.raised_cosine(hop)
y,seg=params.framewise_forward(torch.from_numpy(e).cuda(),torch.from_numpy(fr).cuda(),plan)
ry,rseg=oracle.framewise_forward(e.astype(np.float64),fr.astype(np.float64),hop)
seg=seg.cpu().numpy()[0] if seg.dim()==3 else seg.cpu().numpy()
print('seg shape',seg.shape, 'ref', np.asarray(rseg).shape)
rs=np.asarray(rseg)
for f in range(seg.shape[0]):
    err=np.abs(seg[f]-rs[f]).max()/max(np.abs(rs[f]).max(),1e-8)
    if err>1e-5: print('frame',f,'err',err, 'argmax', np.abs(seg[f]-rs[f]).argmax())
y=y.cpu().numpy()
print('y err', oracle.gradcheck_error(y,ry), 'worst t', np.abs(y-ry).argmax(), 'T', len(y))
# fp32 reference (C restatement in fp32) vs fp64
ry32,_=oracle.framewise_forward(e,fr,hop)
print('ref fp32 err', oracle.gradcheck_error(ry32,ry))
