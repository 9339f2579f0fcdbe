"""oracle — plain CPU oracle for the Flux hot path (arXiv 2508.19078).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2508_19078_b200``) never imports it and
shares no code with it.

Everything is computed in fp64 by ``oracle/oracle.c`` (see its header for the
paper passage each function follows); this module only marshals numpy arrays.

Function → paper passage (P:N = PAPER.md line N; R# = DESIGN.md §2 reading):
  quantize / pack_int4 ........ O1  P:556-565; R1
  router ...................... O2  P:217-220; R2
  permute ..................... O3  P:579-584 (D_e); O8 P:296-298 (hist); R3
  moe_tokens .................. O4-O6 P:196-220; R4-R7
  layer_budget ................ O9  eq.(1); R9
  merge ....................... O10 eq.(2); R10
  profile_tokens .............. O7  layer chaining x_{l+1} = y_l (R7) over the
                                    synthetic model of ``synth`` (inputs only)
Parity pins: tests/test_oracle_*.py.  Unpinned functions: none.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int


def build():
    src = os.path.join(_HERE, "oracle.c")
    out = os.path.join(_HERE, "liboracle.so")
    # no -ffast-math, no FMA contraction: every fp operation is the IEEE one written in the source
    cmd = f"gcc -O2 -std=c11 -fopenmp -fPIC -shared -ffp-contract=off -fno-fast-math -o {out} {src} -lm"
    if os.system(cmd) != 0:
        raise RuntimeError("oracle build failed: " + cmd)


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(os.path.join(_HERE, "oracle.c")):
            build()
        L = ctypes.CDLL(path)
        L.orc_bf16_round.argtypes = [ctypes.c_double]
        L.orc_bf16_round.restype = ctypes.c_double
        L.orc_bf16_round_array.argtypes = [_I64, _P, _P]
        L.orc_quantize.argtypes = [_I, _I64, _I64, _I64, _P, _P, _P]
        L.orc_quantize.restype = _I
        L.orc_pack_int4.argtypes = [_I64, _I64, _P, _P]
        L.orc_pack_int2.argtypes = [_I64, _I64, _P, _P]
        L.orc_attention_hist.argtypes = [_I64, _I, _P, _P, _P]
        L.orc_attention_hist.restype = None
        L.orc_router.argtypes = [_I64, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P]
        L.orc_router.restype = _I
        L.orc_permute.argtypes = [_I64, _I, _I, _P, _P, _P, _P, _P]
        L.orc_moe_tokens.argtypes = [_I64, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I]
        L.orc_moe_tokens.restype = _I
        L.orc_compact_tokens.argtypes = [_I64, _I, _I, _I, _I, _I, _I, _I] + [_P] * 17
        L.orc_layer_budget.argtypes = [_I, _I, _P, _I64, _I64, _P, _P, _P, _P]
        L.orc_layer_budget.restype = _I64
        L.orc_merge.argtypes = [_I, _I64, _P, _P, _P, _I, _P, _P]
        L.orc_merge.restype = _I
        _lib = L
    return _lib


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ------------------------------------------------------------------------------------------
def bf16_round(v):
    """Round real numbers to the nearest bf16 value (ties to even), returned as float64."""
    a = _c(v, np.float64)
    out = np.empty_like(a)
    lib().orc_bf16_round_array(a.size, a.ctypes.data, out.ctypes.data)
    return out


def quantize(w, wbits: int, group_size: int):
    """O1: w [R][K] (float32 values) -> (q int8 [R][K] unpacked, s float32 [R][K/g]). group_size 0 = per row."""
    w = _c(w, np.float32)
    R, K = w.shape
    g = group_size or K
    q = np.empty((R, K), np.int8)
    s = np.empty((R, K // g), np.float32)
    if lib().orc_quantize(wbits, g, R, K, w.ctypes.data, q.ctypes.data, s.ctypes.data):
        raise ValueError("bad quantization arguments")
    return q, s


def pack_int2(q):
    """Canonical INT2 storage: four codes per byte, element k in bits 2·(k mod 4)."""
    q = _c(q, np.int8)
    R, K = q.shape
    out = np.empty((R, K // 4), np.uint8)
    lib().orc_pack_int2(R, K, q.ctypes.data, out.ctypes.data)
    return out


def pack(q, wbits: int):
    """Canonical storage of codes at a bit level (INT8 unpacked)."""
    return pack_int2(q) if wbits == 2 else pack_int4(q) if wbits == 4 else _c(q, np.int8)


def pack_int4(q):
    q = _c(q, np.int8)
    R, K = q.shape
    out = np.empty((R, K // 2), np.uint8)
    lib().orc_pack_int4(R, K, q.ctypes.data, out.ctypes.data)
    return out


def router(x, wr, k: int, norm: int):
    """O2: x [T][H], wr [E][H] (real) -> (z [T][E], ids [T][k] int32, w [T][k], margin [T])."""
    x = _c(x, np.float64)
    wr = _c(wr, np.float64)
    T, H = x.shape
    E = wr.shape[0]
    z = np.empty((T, E))
    ids = np.empty((T, k), np.int32)
    w = np.empty((T, k))
    m = np.empty(T)
    if lib().orc_router(T, H, E, k, norm, x.ctypes.data, wr.ctypes.data, z.ctypes.data, ids.ctypes.data,
                        w.ctypes.data, m.ctypes.data):
        raise ValueError("bad router arguments")
    return z, ids, w, m


def permute(ids, E: int):
    """O3: ids [T][k] (-1 = empty pick) -> (hist [E] int64, offsets [E+1], token_index [offsets[E]], inv_pos [T][k])."""
    ids = _c(ids, np.int32)
    T, k = ids.shape
    hist = np.zeros(E, np.int64)
    off = np.empty(E + 1, np.int64)
    ti = np.empty(T * k, np.int64)
    inv = np.empty((T, k), np.int64)
    lib().orc_permute(T, E, k, ids.ctypes.data, hist.ctypes.data, off.ctypes.data, ti.ctypes.data, inv.ctypes.data)
    return hist, off, ti[:off[E]], inv


class _Expert(ctypes.Structure):
    _fields_ = [("q_gate", _P), ("q_up", _P), ("q_down", _P), ("s_gate", _P), ("s_up", _P), ("s_down", _P)]


class QExpert:
    """Quantized SwiGLU expert: q int8 [rows][K] unpacked + fp32 scales [rows][K/g]."""

    def __init__(self, q_gate, s_gate, q_up, s_up, q_down, s_down):
        self.arrs = [_c(q_gate, np.int8), _c(q_up, np.int8), _c(q_down, np.int8), _c(s_gate, np.float32),
                     _c(s_up, np.float32), _c(s_down, np.float32)]

    def struct(self):
        return _Expert(*[a.ctypes.data for a in self.arrs])


def moe_tokens(x, wr, experts, shared, *, k: int, group_size: int, norm: int, residual=None, with_cond=False,
               exact_dequant=False):
    """O2+O4-O6 for independent tokens of one layer. Returns (y, ids, w, z, margin), plus cond when
    with_cond: cond[t][h] = |r| + |sh| + Σ_j w_j|o_j| (the magnitude of the terms of the O6 sum) and
    dmag[t][h] = Σ_j w_j max_f |a_jf·ŵd_hf| + max_f |a_sh,f·ŵsh_hf| (the largest down-projection term).
    residual: [n][H] real values (e.g. zeros: y is the MoE branch alone) or None (r = x, R6).
    exact_dequant: grouped codes dequantized as ŵ = q·s exactly instead of reading R1b's
    bf16(q·bf16(s)); only for showing that R1b does not decide parity."""
    x = _c(x, np.float64)
    r = None if residual is None else _c(residual, np.float64)
    if r is not None and r.shape != x.shape:
        raise ValueError("residual must have the shape of x")
    wr = _c(wr, np.float64)
    n, H = x.shape
    E = wr.shape[0]
    F = experts[0].arrs[0].shape[0]
    Fs = shared.arrs[0].shape[0] if shared is not None else 0
    arr = (_Expert * E)(*[e.struct() for e in experts])
    sh = ctypes.pointer(shared.struct()) if shared is not None else None
    y = np.empty((n, H))
    ids = np.empty((n, k), np.int32)
    w = np.empty((n, k))
    z = np.empty((n, E))
    m = np.empty(n)
    cond = np.empty((n, H)) if with_cond else None
    dmag = np.empty((n, H)) if with_cond else None
    rc = lib().orc_moe_tokens(n, H, E, k, F, Fs, group_size, norm, x.ctypes.data, wr.ctypes.data,
                              ctypes.cast(arr, _P), ctypes.cast(sh, _P) if sh is not None else None,
                              r.ctypes.data if r is not None else None, y.ctypes.data, ids.ctypes.data,
                              w.ctypes.data, z.ctypes.data, m.ctypes.data,
                              cond.ctypes.data if cond is not None else None,
                              dmag.ctypes.data if dmag is not None else None, int(bool(exact_dequant)))
    if rc:
        raise RuntimeError(f"orc_moe_tokens failed ({rc})")
    if with_cond:
        return y, ids, w, z, m, cond, dmag
    return y, ids, w, z, m


def compact_tokens(x, wr, remap, gate, up, down, shared=None, *, k: int, norm: int, residual=None,
                   with_cond=False):
    """O11 (NEXT-2): gate re-routing through remap + compact-model forward with full-precision weights.
    gate/up [S][F][H], down [S][H][F]; shared = (gate [Fs][H], up [Fs][H], down [H][Fs]) or None.
    residual / with_cond as in moe_tokens.  Returns (y, ids (slot or -1), w, z, margin[, cond, dmag])."""
    x = _c(x, np.float64)
    r = None if residual is None else _c(residual, np.float64)
    wr = _c(wr, np.float64)
    n, H = x.shape
    Er = wr.shape[0]
    g, u, d = _c(gate, np.float64), _c(up, np.float64), _c(down, np.float64)
    S, F = g.shape[0], g.shape[1]
    if shared is not None:
        sg, su, sd = (_c(a, np.float64) for a in shared)
        Fs = sg.shape[0]
    else:
        sg = su = sd = None
        Fs = 0
    rm = _c(remap, np.int32)
    y = np.empty((n, H))
    ids = np.empty((n, k), np.int32)
    w = np.empty((n, k))
    z = np.empty((n, Er))
    m = np.empty(n)
    cond = np.empty((n, H)) if with_cond else None
    dmag = np.empty((n, H)) if with_cond else None
    p = lambda a: None if a is None else a.ctypes.data  # noqa: E731
    rc = lib().orc_compact_tokens(n, H, Er, k, S, F, Fs, norm, x.ctypes.data, wr.ctypes.data, rm.ctypes.data,
                                  g.ctypes.data, u.ctypes.data, d.ctypes.data, p(sg), p(su), p(sd), p(r), y.ctypes.data,
                                  ids.ctypes.data, w.ctypes.data, z.ctypes.data, m.ctypes.data, p(cond), p(dmag))
    if rc:
        raise ValueError(f"orc_compact_tokens failed ({rc})")
    if with_cond:
        return y, ids, w, z, m, cond, dmag
    return y, ids, w, z, m


def attention_hist(ids, attn, E: int, A=None):
    """O13: A [E] int64 += Σ over live picks of RNE(a_t·2^24) (α_e = A_e / (2^24·T) = f_e·ā_e)."""
    ids = _c(ids, np.int32)
    T, k = ids.shape
    a = _c(attn, np.float32)
    A = np.zeros(E, np.int64) if A is None else A
    lib().orc_attention_hist(T, k, ids.ctypes.data, a.ctypes.data, A.ctypes.data)
    return A


def layer_budget(hist, T: int, B_non: int, n_non=None):
    """O9, eq.(1): hist [L][E] int64 -> (C [L] int32, b [L], v [L], overrun)."""
    hist = _c(hist, np.int64)
    L, E = hist.shape
    C = np.empty(L, np.int32)
    b = np.empty(L)
    v = np.empty(L)
    nn = _c(n_non, np.int32) if n_non is not None else None
    over = lib().orc_layer_budget(L, E, hist.ctypes.data, T, B_non, nn.ctypes.data if nn is not None else None,
                                  C.ctypes.data, b.ctypes.data, v.ctypes.data)
    return C, b, v, int(over)


def merge(experts, cluster_of, alpha, n_clusters: int):
    """O10, eq.(2): experts [E][numel] real -> (merged [C][numel] fp64 unrounded, remap [E])."""
    ex = _c(experts, np.float64)
    E, numel = ex.shape
    co = _c(cluster_of, np.int32)
    al = _c(alpha, np.float64)
    out = np.empty((n_clusters, numel))
    remap = np.empty(E, np.int32)
    if lib().orc_merge(E, numel, ex.ctypes.data, co.ctypes.data, al.ctypes.data, n_clusters, out.ctypes.data,
                       remap.ctypes.data):
        raise ValueError("bad merge arguments (empty cluster or cluster id out of range)")
    return out, remap
