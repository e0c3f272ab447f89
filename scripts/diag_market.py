import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from paper_2501_10709_b200 import fin
from oracle import market as om
from synth import market as sm
for K, rows, mag, seed in [(4, 65, 0.0, 0), (30, 200, 0.01, 77), (7, 33, 0.05, 5)]:
    m = sm.stock_market(K=K, rows=rows, seed=seed + 1)
    x = np.stack([m.open_all, m.high_all, m.low_all, m.close_all, m.volume_all], axis=1).astype(np.float32)
    ind = list(om.INDICATORS); I = len(ind)
    mk = torch.zeros((rows, 2 + I, K), dtype=torch.float32, device='cuda')
    raw = torch.zeros((I, K, rows), dtype=torch.float64, device='cuda')
    fin.fin_market_prepare(torch.from_numpy(x).cuda(), sm.WARMUP_DAYS, ind, mk, raw, magnitude=mag, seed=seed)
    o_mk, o_raw = om.prepare_stock_market(x, sm.WARMUP_DAYS, ind, magnitude=mag, seed=seed)
    g = raw.cpu().numpy(); o = np.transpose(o_raw, (1, 2, 0))
    for i, n in enumerate(ind):
        d = np.abs(g[i] - o[i]); r = d / np.maximum(np.abs(o[i]), 1e-300)
        print(K, rows, n, int((g[i] != o[i]).sum()), float(d.max()), float(r.max()))
    gm = mk.cpu().numpy()
    print('market mismatches per channel', [(int((gm[:, c] != o_mk[:, c]).sum())) for c in range(2 + I)])
