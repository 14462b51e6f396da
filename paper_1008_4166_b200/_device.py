"""Device-memory plumbing via torch (allocation, copies, streams only)."""

import numpy as np

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def is_cuda_tensor(x):
    try:
        t = torch()
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, t.Tensor) and x.is_cuda


def empty_colmajor(m, n, dtype, device):
    """m x n tensor with column-major storage (stride (1, m))."""
    return torch().empty((n, m), dtype=dtype, device=device).t()


def is_colmajor(t):
    return t.dim() == 2 and t.stride(0) == 1 and t.stride(1) >= max(1, t.shape[0])


def as_device_colmajor(G, device=None):
    """(tensor with stride (1, m), m, n) on the GPU; copies if needed."""
    t = torch()
    if is_cuda_tensor(G):
        if G.dtype not in (t.float64, t.complex128):
            raise ValueError("G must be float64 or complex128")
        if not (is_colmajor(G) and G.stride(1) == G.shape[0]):
            G = G.t().contiguous().t()
        return G, G.shape[0], G.shape[1]
    A = np.asarray(G)
    if A.ndim != 2:
        raise ValueError("expected a 2-d array")
    A = np.asfortranarray(A, dtype=np.complex128 if np.iscomplexobj(A) else np.float64)
    dev = t.device("cuda", t.cuda.current_device()) if device is None else device
    T = t.from_numpy(A.T.copy()).to(dev)  # (n, m) rows are the columns
    return T.t(), A.shape[0], A.shape[1]


def to_host(U):
    """Column-major device tensor -> Fortran-ordered numpy array."""
    return np.asfortranarray(U.t().contiguous().cpu().numpy().T)


def signs_to_device(signs, n, device):
    s = np.ascontiguousarray(np.asarray(signs).reshape(-1), dtype=np.int8)
    if s.size != n:
        raise ValueError(f"sign vector length {s.size} != column count {n}")
    return torch().from_numpy(s).to(device)


def pinned_host_colmajor(m, n, np_dtype):
    """Fresh m x n column-major numpy array in page-locked host memory
    (torch's caching host allocator: after the first call the pages are
    recycled from freed results, so the device->host copy runs at full
    link speed with no page faults).  The array keeps its storage alive."""
    import numpy as np
    t = torch()
    tdt = {np.dtype(np.float64): t.float64, np.dtype(np.complex128): t.complex128}[np.dtype(np_dtype)]
    buf = t.empty((n, m), dtype=tdt, pin_memory=True)
    return buf.numpy().T
