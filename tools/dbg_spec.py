import sys; sys.path.insert(0,'.')
import numpy as np, torch, oracle, synth, paper_1103_4881_b200 as ds
sys.path.insert(0,'tests')
from test_spec_kernel_gpu import HALO, _stage
for (W,H,ch,chroma,n) in [(352,288,3,1,7),(352,288,3,1,1),(352,288,3,0,2),(176,144,1,1,2)]:
    d = ds.Downscaler(W,H,ch,chroma=chroma,spec=ds.make_spec(h=HALO[0],v=HALO[1],chroma=chroma)); d.set_kernel(ds.DS_KERNEL_FUSED_GENERAL)
    fr = synth.random_frames(77,3,n,W,H,ch,chroma)
    y = d(torch.from_numpy(fr).cuda()).cpu().numpy()
    want = oracle.execute_frames(fr,W,H,ch,chroma,_stage(HALO[0]),_stage(HALO[1]))
    print(W,H,ch,chroma,n,'variant',d.last_variant(), d.launch_info(n))
    for f in range(n):
        planes = oracle.split_planes(y[f],W,H,ch,chroma,out=True,h=_stage(HALO[0]),v=_stage(HALO[1]))
        wp = oracle.split_planes(want[f],W,H,ch,chroma,out=True,h=_stage(HALO[0]),v=_stage(HALO[1]))
        for p,(a,b) in enumerate(zip(planes,wp)):
            bad=np.argwhere(a!=b)
            if len(bad): print(' frame',f,'plane',p,'shape',a.shape,'nbad',len(bad),'rows',sorted(set(bad[:,0].tolist()))[:12],'cols',sorted(set(bad[:,1].tolist()))[:8])
