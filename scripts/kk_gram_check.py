"""Spot-check the device kernel matrix at scale against f64 host values (diagnostic)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2501_05587_b200.kernels import KernelSpec, kernel_matrix, padded_ld
n, d = int(sys.argv[1]), int(sys.argv[2])
fam = sys.argv[3]
g = torch.Generator(device="cuda").manual_seed(0)
P = torch.rand((n, d), device="cuda", generator=g)
spec = KernelSpec(family=fam, gamma=1.0 / d, coef=1.0, degree=2)
K = torch.empty((n, padded_ld(n)), device="cuda")
kernel_matrix(P[:512].contiguous(), spec)
for rep in range(3):
    K.fill_(float("nan"))
    torch.cuda.synchronize(); t0 = time.perf_counter()
    kernel_matrix(P, spec, out=K)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    Ph = P.double().cpu().numpy()
    rng = np.random.default_rng(rep)
    i = rng.integers(0, n, 20000); j = rng.integers(0, n, 20000)
    b = (Ph[i] * Ph[j]).sum(1)
    if fam == "polynomial":
        ref = (b / d + 1.0) ** 2
    else:
        sq = (Ph[i] ** 2).sum(1) + (Ph[j] ** 2).sum(1) - 2 * b
        ref = np.exp(np.maximum(-sq / d, -88.0)); ref[i == j] = 1.0
    got = K[torch.from_numpy(i).cuda(), torch.from_numpy(j).cuda()].double().cpu().numpy()
    print(f"rep {rep}: {dt*1e3:.1f} ms, nan entries {int(torch.isnan(K[:, :n]).sum())}, max rel err {np.max(np.abs(got-ref)/np.abs(ref)):.2e}")
