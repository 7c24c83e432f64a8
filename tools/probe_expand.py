import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2107_01715_b200 as P
from synth.inputs import config
cfg = config("C3")
h = P.Handle.from_config(cfg)
for n in (2,):
    roots = torch.from_numpy(cfg.roots(n).view(np.uint8).reshape(n, -1).copy()).cuda()
    st, cum = h.expand(roots, n, 1, np.float32(cfg.gamma))
    torch.cuda.synchronize()
    print(torch.cuda.synchronize(), "err:", P.lib().bcts_last_error(h._h))
    s = st.cpu().numpy().reshape(n * 18, -1)
    print("zero children:", [i for i in range(n * 18) if not s[i].any()])
    print("cum:", cum.cpu().numpy())
    print("keys:", [hex(int(x)) for x in s[:, :8].copy().view(np.uint64).ravel()])
