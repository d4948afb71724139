import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2408_12479_b200 import emfgpu as G, inputs as I
for (n, p, model, strat, amp) in ((16, 2, "fiber", "none", 0.05), (16, 2, "cnh", "none", 0.05), (16, 2, "fiber", "none", 0.0), (16, 3, "fiber", "none", 0.05), (32, 2, "fiber", "none", 0.05)):
    lev = G.FeLevel(n, p=p, map_param=(amp,))
    prm = G.MaterialParams(mu=1.0, lam=10.0, kappa_b=50.0)
    op = G.ElasticOperator(lev, model, prm, strat, 64)
    op.update_linearization(I.make_u0(n, n, n, p, amp=0.05))
    x = torch.tensor(I.make_v(lev.n_dofs), device="cuda")
    y1 = torch.empty_like(x); y2 = torch.empty_like(x)
    op.apply_elements(x, 0, n); op.apply_nodes(x, y2, 0, n * p)
    bad = []
    for it in range(20):
        y1.fill_(float("nan"))
        op.apply_tangent_device(x, y1); torch.cuda.synchronize()
        d = (y1 != y2).nonzero()
        bad.append(int(d.numel()))
    print(n, p, model, amp, "mismatching entries per run:", bad, flush=True)
    if bad[-1]:
        idx = d[:10, 0].cpu().numpy()
        print("  first idx", idx, "nodes", idx // 3, y1[d[:5,0]].cpu().numpy(), y2[d[:5,0]].cpu().numpy())
