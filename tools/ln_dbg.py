import sys, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_2104_05755_b200 as tpp
from gpu_util import to_dev, to_host
sys.path.insert(0, "/root/repo/oracle")
import tpp_oracle as O
rng = np.random.default_rng(21)
for (n_b, m_b, bn, bm) in ((4, 16, 32, 64), (700, 1, 32, 64), (5, 5, 48, 64)):
    x = O.fp32_to_bf16_rne(rng.normal(0, 1, (n_b, m_b, bn, bm)).astype(np.float32) + 0.3)
    gam = (1 + 0.1 * rng.standard_normal(m_b * bm)).astype(np.float32)
    bet = (0.1 * rng.standard_normal(m_b * bm)).astype(np.float32)
    mean = torch.empty(n_b * bn, dtype=torch.float32, device="cuda"); var = torch.empty_like(mean)
    out = tpp.layernorm_blocked(to_dev(x), n_b, m_b, bn, bm, 1e-5, to_dev(gam), to_dev(bet), mean_out=mean, var_out=var)
    logical = O.bf16_to_fp32(x).transpose(0, 2, 1, 3).reshape(n_b * bn, m_b * bm)
    ref, mu, vr = O.layernorm(logical, gam[None, :], bet[None, :], 1e-5)
    ref = O.fp32_to_bf16_rne(ref.reshape(n_b, bn, m_b, bm).transpose(0, 2, 1, 3)).reshape(-1)
    got = to_host(out)
    bad = np.nonzero(got != ref)[0]
    print((n_b, m_b, bn, bm), "mismatch", len(bad), "of", got.size, "mean ok", np.array_equal(to_host(mean), mu.astype(np.float32)))
    if len(bad):
        idx = np.unravel_index(bad[:10], (n_b, m_b, bn, bm)); print(list(zip(*idx)))
        print(got[bad[:5]], ref[bad[:5]])
