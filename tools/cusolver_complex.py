"""the complex-Hermitian route on the B200 box called through
cuSOLVER's 64-bit API directly (ctypes on the bundled libcusolver), beside this repo's skew
solver on the same seeded matrix.  A library comparison system, never the product path.

The paper's comparison (Tables 1-2 at P:819-824) is its real
skew solver against the complex Hermitian solver on H = -iA (A z = i lam z <=> H z = lam z).
The spectrum of H is {+-lam_k}; the top n/2 eigenpairs of H are the skew solver's nev = n/2
pairs (z_k), and the other half are their conjugates (z-bar_k for -lam_k), so one
skew solve with nev = n/2 answers both rows:
  * 50 %:  the top n/2 eigenpairs of H (cusolverDnXsyevdx, index range  vs skew nev = n/2
           il = n/2+1 .. iu = n)
  * 100 %: all n eigenpairs of H (cusolverDnXsyevd, complex128)        vs skew nev = n/2
           (+ the conjugate half, free: expand_half_spectrum)
  * eigenvalues only (jobz = NOVECTOR, all and top half)               vs skew_eigvals
Times are CUDA-event device times with inputs resident in HBM (best of --reps for the skew
side, one run for the complex side).  A cuSOLVER failure (status / workspace / memory) is
recorded in the output line, never extrapolated.

python tools/cusolver_complex.py --n 8192 16384 32768
"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1912_04062_b200 as sk  # noqa: E402
import skewgen  # noqa: E402

CUDA_R_64F, CUDA_C_64F = 1, 5
MODE_NOVECTOR, MODE_VECTOR = 0, 1
RANGE_ALL, RANGE_I = 1001, 1002
FILL_LOWER = 0
_vp, _i64, _sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_size_t


def _libcusolver():
    import nvidia.cusolver as ncs
    d = os.path.join(list(ncs.__path__)[0], "lib")
    return ctypes.CDLL(os.path.join(d, "libcusolver.so.11"))


class CuSolver:
    def __init__(self, stream):
        self.L = L = _libcusolver()
        self.h, self.p = _vp(), _vp()
        assert L.cusolverDnCreate(ctypes.byref(self.h)) == 0
        assert L.cusolverDnSetStream(self.h, _vp(stream)) == 0
        assert L.cusolverDnCreateParams(ctypes.byref(self.p)) == 0
        L.cusolverDnXsyevd_bufferSize.argtypes = [_vp, _vp, ctypes.c_int, ctypes.c_int, _i64, ctypes.c_int, _vp, _i64,
                                                  ctypes.c_int, _vp, ctypes.c_int, ctypes.POINTER(_sz),
                                                  ctypes.POINTER(_sz)]
        L.cusolverDnXsyevd.argtypes = [_vp, _vp, ctypes.c_int, ctypes.c_int, _i64, ctypes.c_int, _vp, _i64,
                                       ctypes.c_int, _vp, ctypes.c_int, _vp, _sz, _vp, _sz, _vp]
        L.cusolverDnXsyevdx_bufferSize.argtypes = [_vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64,
                                                   ctypes.c_int, _vp, _i64, _vp, _vp, _i64, _i64,
                                                   ctypes.POINTER(_i64), ctypes.c_int, _vp, ctypes.c_int,
                                                   ctypes.POINTER(_sz), ctypes.POINTER(_sz)]
        L.cusolverDnXsyevdx.argtypes = [_vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64, ctypes.c_int, _vp,
                                        _i64, _vp, _vp, _i64, _i64, ctypes.POINTER(_i64), ctypes.c_int, _vp,
                                        ctypes.c_int, _vp, _sz, _vp, _sz, _vp]

    def heev(self, H, W, vectors, il=None, iu=None):
        """In place on the column-major complex128 H (n x n); W real (n).  il/iu (1-based,
        ascending) select an index range via Xsyevdx; None = all via Xsyevd.  Returns
        (status string, meig)."""
        L, n = self.L, H.shape[0]
        dws, hws = _sz(0), _sz(0)
        jobz = MODE_VECTOR if vectors else MODE_NOVECTOR
        vl, vu = ctypes.c_double(0.0), ctypes.c_double(0.0)
        meig = _i64(n)
        if il is None:
            st = L.cusolverDnXsyevd_bufferSize(self.h, self.p, jobz, FILL_LOWER, n, CUDA_C_64F, _vp(H.data_ptr()), n,
                                               CUDA_R_64F, _vp(W.data_ptr()), CUDA_C_64F, ctypes.byref(dws),
                                               ctypes.byref(hws))
        else:
            st = L.cusolverDnXsyevdx_bufferSize(self.h, self.p, jobz, RANGE_I, FILL_LOWER, n, CUDA_C_64F,
                                                _vp(H.data_ptr()), n, ctypes.byref(vl), ctypes.byref(vu), il, iu,
                                                ctypes.byref(meig), CUDA_R_64F, _vp(W.data_ptr()), CUDA_C_64F,
                                                ctypes.byref(dws), ctypes.byref(hws))
        if st != 0:
            return f"bufferSize status {st}", 0
        try:
            dbuf = torch.empty(max(dws.value, 1), dtype=torch.uint8, device=H.device)
        except torch.OutOfMemoryError:
            return f"device workspace {dws.value / 2**30:.1f} GiB does not fit", 0
        hbuf = ctypes.create_string_buffer(max(hws.value, 1))
        info = torch.zeros(1, dtype=torch.int32, device=H.device)
        if il is None:
            st = L.cusolverDnXsyevd(self.h, self.p, jobz, FILL_LOWER, n, CUDA_C_64F, _vp(H.data_ptr()), n, CUDA_R_64F,
                                    _vp(W.data_ptr()), CUDA_C_64F, _vp(dbuf.data_ptr()), dws.value, hbuf,
                                    hws.value, _vp(info.data_ptr()))
        else:
            st = L.cusolverDnXsyevdx(self.h, self.p, jobz, RANGE_I, FILL_LOWER, n, CUDA_C_64F, _vp(H.data_ptr()), n,
                                     ctypes.byref(vl), ctypes.byref(vu), il, iu, ctypes.byref(meig), CUDA_R_64F,
                                     _vp(W.data_ptr()), CUDA_C_64F, _vp(dbuf.data_ptr()), dws.value, hbuf,
                                     hws.value, _vp(info.data_ptr()))
        torch.cuda.synchronize()
        if st != 0 or int(info.item()) != 0:
            return f"status {st} info {int(info.item())}", 0
        return "ok", meig.value


def timed(fn, reps):
    best, out = None, None
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    return best, out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--n", type=int, nargs="+", default=[8192, 16384, 32768])
    p.add_argument("--reps", type=int, default=2)
    a = p.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cs = CuSolver(torch.cuda.current_stream().cuda_stream)
    ctx = sk.Context()
    for n in a.n:
        row = {"n": n, "complex_system": "cuSOLVER 64-bit API (cusolverDnXsyevd / cusolverDnXsyevdx), complex128"}
        A0 = torch.empty((n, n), dtype=torch.float64, device=dev).t()   # column-major lower
        skewgen.random_skew_lower_device(A0, n, n, torch.cuda.current_stream().cuda_stream)
        A = torch.empty_like(A0.t()).t()

        def skew(nev, vectors=True):
            def f():
                A.copy_(A0)
                if vectors:
                    return sk.skew_eig(A, nev, ctx=ctx, overwrite_a=True)
                return sk.skew_eigvals(A, nev, ctx=ctx, overwrite_a=True)
            return f

        tsk, (lam, Zre, Zim) = timed(skew(n // 2), a.reps)
        lam = lam.clone()
        del Zre, Zim
        tev, _ = timed(skew(n // 2, vectors=False), a.reps)
        row.update(skew_half_spectrum_s=tsk / 1e3, skew_eigvals_s=tev / 1e3)
        del A
        torch.cuda.empty_cache()
        nA = None
        for tag, vectors, rng in (("all", True, None), ("half", True, (n // 2 + 1, n)),
                                  ("eigvals", False, None), ("half_eigvals", False, (n // 2 + 1, n))):
            L = torch.tril(A0, -1)
            H = ((-1j) * (L - L.t()).to(torch.complex128)).t().contiguous().t()   # Hermitian -iA, column-major
            del L
            if nA is None:
                nA = torch.linalg.norm(H).item()
            W = torch.zeros(n, dtype=torch.float64, device=dev)
            try:
                t, (status, meig) = timed(lambda: cs.heev(H, W, vectors, *(rng or (None, None))), 1)
            except torch.OutOfMemoryError as e:
                t, status, meig = None, "out of memory: " + str(e).splitlines()[0][:120], 0
            row[f"complex_{tag}_s"] = t / 1e3 if (t is not None and status == "ok") else None
            if status != "ok":
                row[f"complex_{tag}_error"] = status
            else:
                wtop = torch.flip(W[:n] if rng is None else W[:meig], [0])[: n // 2]   # descending positive half
                row[f"max_dlam_{tag}_over_normA"] = (lam[: len(wtop)] - wtop).abs().max().item() / nA
            del H, W
            torch.cuda.empty_cache()
        for tag, ref in (("all", "skew_half_spectrum_s"), ("half", "skew_half_spectrum_s"),
                         ("eigvals", "skew_eigvals_s"), ("half_eigvals", "skew_eigvals_s")):
            if row.get(f"complex_{tag}_s"):
                row[f"speedup_{tag}"] = row[f"complex_{tag}_s"] / row[ref]
        print(json.dumps(row), flush=True)
        del A0
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
