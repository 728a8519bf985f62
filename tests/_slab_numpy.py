"""Plain numpy stand-in for the four slab phases (TEST INFRASTRUCTURE ONLY).

Lets the CPU tests run paper_2504_05808_b200/slab.py's real exchange code over gloo without a
GPU.  Each phase computes, by brute force on the small test volumes, what the corresponding
C-ABI phase computes (include/fastrs.h "multi-GPU z-slab path"), with the same windowing
semantics: a phase sees only the slices it is given, so a too-small halo makes the result
wrong, which is what the tests would catch.  No pruning (every object element is a ball
centre); plain per-run minima for the separable passes.
"""
from __future__ import annotations

import math

import numpy as np
import torch

INF = (1 << 30) - 1
BIT_Z = 1 << 30


def _runs(v):
    """[(start, end)] of maximal runs of equal values in a 1D array."""
    out, a = [], 0
    for i in range(1, len(v) + 1):
        if i == len(v) or v[i] != v[a]:
            out.append((a, i - 1))
            a = i
    return out


def _line_min(g, a, b, site_lo, site_hi):
    """Per-run squared distance: min over q in [a,b] of g(q) + (p-q)^2, plus the run-end sites."""
    res = np.zeros(b - a + 1, np.int64)
    for p in range(a, b + 1):
        best = INF
        for q in range(a, b + 1):
            if g[q] < INF:
                best = min(best, int(g[q]) + (p - q) ** 2)
        if site_lo:
            best = min(best, (p - a + 1) ** 2)
        if site_hi:
            best = min(best, (b + 1 - p) ** 2)
        res[p - a] = min(best, INF)
    return res


FX_SCALE = 2.0 ** 32  # fixed-point scale of the LT sums (csrc/common.cuh "Accum")


def split_sum(fx: np.ndarray) -> tuple[int, int]:
    """(hi, lo) accumulator words of a sum of fixed-point terms: sum(t >> 32), sum(t & (2^32-1))."""
    return int((fx >> np.uint64(32)).sum(dtype=np.uint64)), int((fx & np.uint64(0xFFFFFFFF)).sum(dtype=np.uint64))


class NumpyPhases:
    def edt_xy(self, labels, below, max_label, flags):
        lab = labels.numpy()
        border = bool(flags & 1)
        nz, Y, X = lab.shape
        g = np.zeros(lab.shape, np.int64)
        for z in range(nz):
            for y in range(Y):
                row = lab[z, y]
                for a, b in _runs(row):
                    if row[a] == 0:
                        continue
                    for p in range(a, b + 1):
                        dl = p - a + 1 if (a > 0 or border) else INF
                        dr = b + 1 - p if (b < X - 1 or border) else INF
                        d = min(dl, dr)
                        g[z, y, p] = INF if d >= INF else d * d
        dxy = np.zeros(lab.shape, np.int64)
        for z in range(nz):
            for x in range(X):
                col = lab[z, :, x]
                for a, b in _runs(col):
                    if col[a] == 0:
                        continue
                    dxy[z, a:b + 1, x] = _line_min(g[z, :, x], a, b, a > 0 or border, b < Y - 1 or border)
        prev = np.empty_like(lab)
        prev[1:] = lab[:-1]
        zflag = np.ones(lab.shape, bool)
        zflag[1:] = lab[1:] != prev[1:]
        if below is not None:
            zflag[0] = lab[0] != below.numpy()
        packed = (dxy | np.where(zflag, BIT_Z, 0)).astype(np.int64)
        m = int(dxy[lab != 0].max()) if (lab != 0).any() else 0
        return torch.from_numpy(packed.astype(np.uint32).view(np.int32)), torch.tensor([m], dtype=torch.int32)

    def edt_z(self, packed_ext, own_lo, own_hi, z_ext0, Z, flags):
        w = packed_ext.numpy().view(np.uint32).astype(np.int64)
        border = bool(flags & 1)
        g = w & INF
        start = (w & BIT_Z) != 0
        n, Y, X = w.shape
        d = np.zeros((own_hi - own_lo, Y, X), np.int64)
        for y in range(Y):
            for x in range(X):
                a = 0
                for t in range(1, n + 1):
                    if t == n or start[t, y, x]:
                        b = t - 1
                        if g[a, y, x] != 0 and b >= own_lo and a < own_hi:
                            # a site below the run: the element before a exists inside the buffer,
                            # or a is the global start with the border flag
                            lo_site = (a > 0 and start[a, y, x]) or (z_ext0 + a == 0 and border)
                            hi_site = (b + 1 < n) or (z_ext0 + n == Z and border)
                            vals = _line_min(g[:, y, x], a, b, lo_site, hi_site)
                            for p in range(max(a, own_lo), min(b, own_hi - 1) + 1):
                                d[p - own_lo, y, x] = vals[p - a]
                        a = t
        obj = d[d > 0]
        m = int(obj.max()) if obj.size else 0
        return torch.from_numpy(d.astype(np.int32)), torch.tensor([m], dtype=torch.int32)

    def reduce(self, labels, d_ext, own_lo, own_hi, Z, dmax, max_label, flags):
        lab = labels.numpy()
        D = d_ext.numpy().astype(np.int64)
        n, Y, X = D.shape
        lt2 = np.zeros((own_hi - own_lo, Y, X), np.int64)
        zz, yy, xx = np.nonzero(D)
        for cz, cy, cx in zip(zz, yy, xx):
            r2 = D[cz, cy, cx] - 1
            r = math.isqrt(r2)
            for z in range(max(own_lo, cz - r), min(own_hi, cz + r + 1)):
                for y in range(max(0, cy - r), min(Y, cy + r + 1)):
                    rem = r2 - (z - cz) ** 2 - (y - cy) ** 2
                    if rem < 0:
                        continue
                    w = math.isqrt(rem)
                    sl = lt2[z - own_lo, y, max(0, cx - w):min(X, cx + w + 1)]
                    np.maximum(sl, D[cz, cy, cx], out=sl)
        fx = np.rint(np.sqrt(lt2.astype(np.float64)) * FX_SCALE).astype(np.uint64)
        shell = D[own_lo:own_hi] == 1
        part = {k: np.zeros(max_label, np.uint64) for k in ("vol", "n_shell")}
        part.update({k: np.zeros(2 * max_label, np.uint64) for k in ("sum_lt", "sum_shell_lt")})
        part["max_lt2"] = np.zeros(max_label, np.int64)
        for k in range(1, max_label + 1):
            m = lab == k
            if not m.any():
                continue
            part["vol"][k - 1] = m.sum()
            part["n_shell"][k - 1] = (m & shell).sum()
            part["sum_lt"][k - 1], part["sum_lt"][max_label + k - 1] = split_sum(fx[m])
            part["sum_shell_lt"][k - 1], part["sum_shell_lt"][max_label + k - 1] = split_sum(fx[m & shell])
            part["max_lt2"][k - 1] = lt2[m].max()
        out = {k: torch.from_numpy(v.view(np.int64).copy()) for k, v in part.items() if k != "max_lt2"}
        out["max_lt2"] = torch.from_numpy(part["max_lt2"].astype(np.int32))
        return out

    def metrics(self, part, nscale, dmax, stats):
        vol = part["vol"].numpy().view(np.uint64).astype(np.float64)
        nsh = part["n_shell"].numpy().view(np.uint64).astype(np.float64)
        M = vol.shape[0]

        def total(k):
            w = part[k].numpy().view(np.uint64).astype(np.float64)
            return w[:M] + w[M:] / FX_SCALE

        sm, ss = total("sum_lt"), total("sum_shell_lt")
        mx = np.sqrt(part["max_lt2"].numpy().astype(np.float64))
        with np.errstate(invalid="ignore", divide="ignore"):
            a = sm / vol
            c = 3 * vol / (4 * math.pi * a * a)
            q = np.minimum(a, c) / np.maximum(a, c)
            e = np.sqrt(1 - q * q)
            obl = 2 * math.pi * a * a * (1 + q * q * np.arctanh(e) / e)
            pro = 2 * math.pi * a * a * (1 + np.arcsin(e) / (q * e))
            area = np.where(e == 0, 4 * math.pi * a * a, np.where(c < a, obl, pro))
            sph = np.cbrt(36 * math.pi * vol * vol) / area
            rnd = (ss / nsh) / mx
        sph[vol == 0] = np.nan
        rnd[vol == 0] = np.nan
        res = {"sphericity": torch.from_numpy(sph), "roundness": torch.from_numpy(rnd)}
        if stats:
            res["volume"] = torch.from_numpy(vol.astype(np.int64))
            res["n_shell"] = torch.from_numpy(nsh.astype(np.int64))
            res["max_lt2"] = part["max_lt2"].clone()
        return res

    def edge(self, labels, max_label, skip_zlo, skip_zhi):
        """Labels on the slab's faces that are faces of the volume (brute force)."""
        lab = labels.numpy()
        out = np.zeros(max_label, np.uint8)
        faces = [lab[:, 0, :], lab[:, -1, :], lab[:, :, 0], lab[:, :, -1]]
        if not skip_zlo:
            faces.append(lab[0])
        if not skip_zhi:
            faces.append(lab[-1])
        for f in faces:
            for L in np.unique(f):
                if 1 <= L <= max_label:
                    out[L - 1] = 1
        return torch.from_numpy(out)

