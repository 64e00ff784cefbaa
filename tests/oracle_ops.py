"""CPU stand-in for parallel.FraqOps (numpy DST + the mode-space oracle) with the same
interface, so the gloo tests exercise the sharding / transpose logic of parallel.py without a GPU.
TEST INFRASTRUCTURE: uses oracle/ (kept out of the product package)."""


class OracleOps:
    """CPU stand-in with the same interface (numpy DST + the mode-space oracle), for the gloo
    tests of the sharding logic.  TEST INFRASTRUCTURE: uses oracle/."""

    def __init__(self, orc, torch):
        self.orc, self.torch = orc, torch
        self.stream = None

    def tensor(self, x):
        return self.torch.as_tensor(x, dtype=self.torch.float64).contiguous()

    def empty(self, *shape):
        return self.torch.empty(*shape, dtype=self.torch.float64)

    def mark(self):
        import time
        return time.perf_counter()

    @staticmethod
    def seconds(a, b):
        return b - a

    def dst2d(self, M, x, inverse):
        import numpy as np
        S = np.sin(np.outer(np.arange(1, M + 1), np.arange(1, M + 1)) * np.pi / (M + 1))
        sc = 1.0 if inverse else (2.0 / (M + 1)) ** 2
        g = x.numpy().reshape(-1, M, M)
        return self.tensor(np.stack([sc * S @ gi @ S for gi in g]).reshape(x.shape))

    def dst_cols(self, M, x, inverse):
        import numpy as np
        S = np.sin(np.outer(np.arange(1, M + 1), np.arange(1, M + 1)) * np.pi / (M + 1))
        sc = 1.0 if inverse else 2.0 / (M + 1)
        return self.tensor(sc * S @ x.numpy().reshape(M, -1)).reshape(x.shape)

    def step(self, alpha1, alpha2, a, t_final, N, scheme, lam, c0, kconf):
        sbd = scheme == "FastSBD"
        tau = t_final / N
        k1 = self.orc.build_kernel_auto(sbd, 1 - alpha1, tau, N)
        k2 = self.orc.build_kernel_auto(sbd, 1 - alpha2, tau, N)
        u, v, secs = self.orc.modal_run(k1, k2, a, tau, N, lam.numpy(), c0[0].numpy(),
                                        c0[1].numpy())
        import numpy as np
        return self.tensor(np.stack([u, v])), secs
