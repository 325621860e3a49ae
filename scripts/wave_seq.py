import sys, json
from pathlib import Path
ROOT = Path('/root/repo'); sys.path.insert(0, str(ROOT))
import numpy as np, torch
import bench
import paper_2602_08798_b200 as api
from paper_2602_08798_b200.backend import GpuContext
from paper_2602_08798_b200.ring import Ring
calls=[]
def wrap(name):
    fn=getattr(Ring,name)
    def w(self,a,*args,**kw):
        extra=''
        if name=='rotate':
            st=np.unique(np.asarray(args[0])); extra=f"steps={st.tolist()[:4]} add={kw.get('add_input', args[2] if len(args)>2 else False)}"
        try: n = len(a)
        except Exception: n = 0
        calls.append(f"{name}[{n}] {extra}")
        return fn(self,a,*args,**kw)
    setattr(Ring,name,w)
for n in ("rotate","mult_cipher","mult_cipher_ext","mult_cipher_ext2","sum","decrypt_start","decrypt_finish","encrypt_batch","mult_plain","add","add_plain","copy"):
    if hasattr(Ring,n): wrap(n)
root, fp, ctxs, caches, chans, rng = bench.build_state(api, GpuContext, 128, 12)
C=GpuContext
toks=[C.w_encrypt([c for c in ctxs for _ in range(3)], np.stack(bench.step_tokens(rng, 12))).handles() for _ in range(3)]
for i in range(3):
    calls.clear()
    cs = api.maybe_refresh_heads(caches, ctxs, chans)
    cs = api.append_token_heads(cs, toks[i][1::3], toks[i][2::3], ctxs)
    api.attention_step_heads(toks[i][0::3], cs, fp, ctxs, chans)
    caches=cs
torch.cuda.synchronize()
print("\n".join(calls))
