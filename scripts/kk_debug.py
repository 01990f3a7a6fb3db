import numpy as np, torch, sys
sys.path.insert(0, '.')
import oracle.kernel_oracle as ko
from paper_2501_05587_b200.kernels import KernelSpec, kernel_matrix
from paper_2501_05587_b200.kkmeans import KernelEngine
n, d, k = 5000, 64, 37
g = np.random.default_rng(n + k)
P = (g.random((n, d)) + g.integers(0, 4, size=(n, 1)) * 0.5).astype(np.float32)
kw = dict(family="polynomial", gamma=1.0 / d, coef=1.0, degree=2)
K64 = ko.apply_kernel(ko.compute_gram(P.astype(np.float64), "gemm"), **kw)
K = kernel_matrix(torch.from_numpy(P).cuda(), KernelSpec(**kw))[:, :n].cpu().numpy()
err = np.abs(K - K64)
print("K max err", err.max(), "at", np.unravel_index(err.argmax(), err.shape), "bad entries", (err > 1e-3).sum())
eng = KernelEngine(P, k, KernelSpec(**kw), max_iters=1)
prev = ko.init_assignments(n, k, 3)
got = eng.step_from(prev)
S_ref = np.zeros((k, n))
for j in range(k):
    S_ref[j] = K64[prev == j].sum(axis=0)
e = np.abs(got["S"] - S_ref)
print("S max err", e.max(), np.unravel_index(e.argmax(), e.shape), "rows bad", np.unique(np.nonzero(e > 1e-2)[0])[:20], "cols bad", np.unique(np.nonzero(e > 1e-2)[1]).size)
print("moved", got["moved"])
