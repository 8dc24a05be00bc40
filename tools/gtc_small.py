import sys; sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2210_09953_b200 as rcq, synth
for (m,n,k,dt) in [(10000,20,40,"f64"),(5000,100,200,"f32")]:
    X = torch.from_numpy(synth.make_X(m, n, 3.0, dt)).cuda()
    plan = rcq.RCholQR(n=n, k=k, dtype=X.dtype, sketch="gaussian")
    try:
        P = plan.sketch(X); torch.cuda.synchronize(); print("ok", m, n, k, dt, float(P[0,0]))
    except Exception as e:
        print("ERR", m, n, k, dt, e)
