"""numpy emulator of the fused kernel's program (test helper, CPU only).

Executes the op records of CompiledCircuit.export() on a full state vector
with the SAME semantics the CUDA kernel implements (desc.h / fused.cu): within
a register stage every "thread" (index with the register bits cleared) holds
2^RB slots; slot p holds the amplitude of logical register index i with
p = L i ^ F, where L is the stage's GF(2) map (register CX gates, never
executed) and F the thread's flip vector (OC_XF).  Ops act on slots
(OC_RD/CD/PH/CXM/PH2/XF), thread phases are applied at the stage end, and the
stage's out vectors (columns of L^-1) plus F route each slot back to its
logical index — exactly the transpose/store addressing of the kernel.
Remaps between segments swap physical positions.  This checks the planner
(scheduling, commutation, fusion, lazy CX, remaps) on a CPU box.
"""

from __future__ import annotations

import numpy as np

RD, CD, PH, CXM, PH2, XF, TPH = range(7)
STAGE = 200


def _bit(idx, q):
    return (idx >> q) & 1


def _swap_positions(psi, n, p1, p2):
    """Exchange physical index bits p1 and p2 (a remap on the full vector)."""
    idx = np.arange(psi.size, dtype=np.int64)
    b1, b2 = _bit(idx, p1), _bit(idx, p2)
    src = idx ^ ((b1 ^ b2) << p1) ^ ((b1 ^ b2) << p2)
    return psi[src]


class _Stage:
    def __init__(self, psi, n, reg_q, out_vec, dtype):
        self.rb = len(reg_q)
        self.reg_q = reg_q
        self.out_vec = out_vec
        self.dtype = dtype
        rmask = 0
        for q in reg_q:
            rmask |= 1 << q
        idx = np.arange(1 << n, dtype=np.int64)
        self.base = idx[(idx & rmask) == 0]  # one entry per thread (its global bits)
        slots = np.arange(1 << self.rb, dtype=np.int64)
        off = np.zeros(slots.size, dtype=np.int64)
        for b, q in enumerate(reg_q):
            off |= _bit(slots, b) << q
        self.off = off
        self.A = psi[self.base[:, None] | off[None, :]].copy()  # [threads, slots]
        self.F = np.zeros(self.base.size, dtype=np.int64)
        self.phase = np.ones(self.base.size, dtype=np.complex128)

    def pred(self, cmask):
        return (self.base & cmask) == cmask

    @staticmethod
    def _par(x):
        x = np.asarray(x, dtype=np.int64)
        r = np.zeros_like(x)
        for b in range(8):
            r ^= (x >> b) & 1
        return r

    def pair_op(self, v, w, m):
        """2x2 on slot pairs {p, p ^ v}; the member with parity(w & p) = 0 is logical |0>;
        threads with parity(w & F) = 1 see X m X."""
        f = self._par(w & self.F).astype(bool)
        lo = [p for p in range(1 << self.rb) if not self._par(w & p)]
        hi = [p ^ v for p in lo]
        m = m.astype(self.dtype)
        mf = m[::-1, ::-1]
        x, y = self.A[:, lo].copy(), self.A[:, hi].copy()
        for mm, sel in ((m, ~f), (mf, f)):
            self.A[np.ix_(sel, lo)] = mm[0, 0] * x[sel] + mm[0, 1] * y[sel]
            self.A[np.ix_(sel, hi)] = mm[1, 0] * x[sel] + mm[1, 1] * y[sel]

    def phase_op(self, w, e, cmask):
        e = np.where(self.pred(cmask), e, 1.0) if cmask else np.full(self.base.size, e)
        f = self._par(w & self.F)
        for p in range(1 << self.rb):
            logical_one = self._par(w & p) ^ f
            mult = np.where(logical_one == 1, e, 1.0).astype(self.dtype)
            self.A[:, p] = self.A[:, p] * mult

    def phase2_op(self, t, c, e):
        ft, fc = _bit(self.F, t), _bit(self.F, c)
        for p in range(1 << self.rb):
            both = (((p >> t) & 1) ^ ft) & (((p >> c) & 1) ^ fc)
            self.A[:, p] = self.A[:, p] * np.where(both == 1, e, 1.0).astype(self.dtype)

    def cxm_op(self, t, c):
        src = self.A.copy()
        for p in range(1 << self.rb):
            q = p ^ ((((p >> c) & 1)) << t)
            self.A[:, q] = src[:, p]
        self.F ^= _bit(self.F, c) << t

    def finish(self, psi):
        self.A *= self.phase[:, None].astype(self.dtype)
        for p in range(1 << self.rb):
            pf = p ^ self.F  # per thread
            lg = np.zeros(self.base.size, dtype=np.int64)  # logical register index L^-1 (p ^ F)
            for j in range(self.rb):
                lg ^= np.where(_bit(pf, j) == 1, self.out_vec[j], 0)
            dst = self.base.copy()
            for b, q in enumerate(self.reg_q):
                dst |= _bit(lg, b) << q
            psi[dst] = self.A[:, p]


def run_program(plan, dtype=np.complex128) -> np.ndarray:
    """Full 2^n state (logical order) after executing `plan` (a CompiledCircuit)."""
    n = plan.n_qubits
    rec, mats = plan.export()
    psi = np.zeros(1 << n, dtype=dtype)
    psi[0] = 1
    idx = np.arange(1 << n, dtype=np.int64)
    remaps = list(plan.remaps)
    last_pass = -1
    st = None
    for r in rec:
        p, s, kind, t, c, cmask, qmask, mi = (int(v) for v in r)
        m = mats[mi]
        if kind == STAGE or kind >= 100:
            if st is not None:
                st.finish(psi)
                st = None
            if p > last_pass + 1:
                # a skipped pass id marks a segment boundary -> apply the remap(s) in between
                for _ in range(p - last_pass - 1):
                    g, loc = remaps.pop(0)
                    for a, b in zip(g, loc):
                        psi = _swap_positions(psi, n, a, b)
            last_pass = p
        if kind == STAGE:
            reg_q = [int(m[b]) for b in range(t)]
            out_vec = [(c >> (6 * j)) & 63 for j in range(t)]
            st = _Stage(psi, n, reg_q, out_vec, dtype)
            continue
        cx = lambda k: complex(m[2 * k], m[2 * k + 1])  # noqa: E731
        if kind in (RD, CD):
            st.pair_op(t, c, np.array([[cx(0), cx(1)], [cx(2), cx(3)]], dtype=np.complex128))
        elif kind == PH:
            st.phase_op(t, cx(0), cmask)
        elif kind == PH2:
            st.phase2_op(t, c, cx(0))
        elif kind == CXM:
            st.cxm_op(t, c)
        elif kind == XF:
            st.F ^= np.where(st.pred(cmask), t, 0)
        elif kind == TPH:
            sel = st.pred(cmask)
            v = np.where((st.base & qmask) != 0, cx(1), cx(0))
            st.phase = np.where(sel, st.phase * v, st.phase)
        elif kind == 100:
            u = np.array([[cx(0), cx(1)], [cx(2), cx(3)]], dtype=np.complex128).astype(dtype)
            sel = (idx & cmask) == cmask
            lo = np.flatnonzero((_bit(idx, t) == 0) & sel)
            hi = lo | (1 << t)
            a, b = psi[lo].copy(), psi[hi].copy()
            psi[lo] = u[0, 0] * a + u[0, 1] * b
            psi[hi] = u[1, 0] * a + u[1, 1] * b
        elif kind == 101:
            sel = (idx & cmask) == cmask
            v = np.where((idx & qmask) != 0, cx(1), cx(0))
            psi[sel] = psi[sel] * v[sel].astype(dtype)
        else:
            raise AssertionError(f"unknown op kind {kind}")
    if st is not None:
        st.finish(psi)
    while remaps:  # trailing remaps (no passes after them)
        g, loc = remaps.pop(0)
        for a, b in zip(g, loc):
            psi = _swap_positions(psi, n, a, b)
    # physical -> logical order: logical qubit q sits at physical position final_map[q]
    fm = np.asarray(plan.final_map)
    if np.any(fm != np.arange(n)):
        src = np.zeros(1 << n, dtype=np.int64)
        for q in range(n):
            src |= _bit(idx, q) << int(fm[q])
        psi = psi[src]
    return psi
