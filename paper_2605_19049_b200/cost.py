"""Algorithmic byte accounting for the KV-buffered GDN decode path.

Two families of formulas:

* ``paper_*`` — the paper's own memory-access model, Table 1 (vanilla LA,
  P:96-113), Table 2 (GDN) and the speedup equations Eq. 6
  (P:157), Eq. 9, Eq. 10 and their exact GDN forms
  (P:436-447).  Single head, FP32 state, FP16 q/k/v/o (reading Z22).
* ``layer_*`` — the bytes THIS build's kernels must move per slot-layer with
  their actual dtypes and record layout: these are
  the numerators of every achieved-GB/s figure bench.py reports.
"""
from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

# ----------------------------------------------------------------- paper model


def paper_table1(form: str, d: int, L: int = 0, m: int = 1):
    """Table 1: (storage, read, write) bytes per token, vanilla LA."""
    if form == "parallel":
        return 4 * L * d, 4 * L * d + 2 * d, 6 * d
    if form == "recurrent":
        return 4 * d * d, 4 * d * d + 6 * d, 4 * d * d + 2 * d
    if form == "chunkwise":
        return (4 * d * d + 4 * m * d,
                Fraction(4 * (m + 1), m) * d * d + 2 * (m + 4) * d,
                Fraction(4 * d * d, m) + 6 * d)
    raise ValueError(form)


def paper_table2(form: str, d: int, L: int = 0, m: int = 1):
    """Table 2: (storage, read, write) bytes per token, GDN."""
    if form == "parallel":
        return 4 * L * d + 2 * L, 4 * L * d + 2 * d + 2 * L + 2, 6 * d + 2
    if form == "recurrent":
        return 4 * d * d, 4 * d * d + 6 * d + 4, 4 * d * d + 2 * d
    if form == "chunkwise":
        return (4 * d * d + 4 * m * d + 2 * m,
                Fraction(4 * (m + 1), m) * d * d + 2 * (m + 4) * d + m + 5,
                Fraction(4 * d * d, m) + 6 * d + 2)
    raise ValueError(form)


def paper_speedup_chunkwise(d, m):
    """Eq. 6: 4(d+1) / (2d + 4d/m + m + 7)."""
    return Fraction(4 * (d + 1)) / (2 * d + Fraction(4 * d, m) + m + 7)


def paper_speedup_chunkwise_gdn(d, m):
    """Exact GDN form."""
    return Fraction(8 * d * d + 8 * d + 4) / (4 * d * d + Fraction(8 * d * d, m) + 2 * m * d + 14 * d + m + 7)


def paper_speedup_verify(d, m):
    """Eq. 9: ((m+1)d + 2m) / (3d + 4m)."""
    return Fraction((m + 1) * d + 2 * m, 3 * d + 4 * m)


def paper_speedup_verify_gdn(d, m):
    """Exact GDN form."""
    return Fraction(4 * (m + 1) * d * d + 8 * m * d + 4 * m, 12 * d * d + 16 * m * d + 8 * m)


def paper_speedup_kv_only(d, m, L):
    """Eq. 10: (d + 2d/m + m/2 + 7/2) / (L + 2)."""
    return (d + Fraction(2 * d, m) + Fraction(m, 2) + Fraction(7, 2)) / (L + 2)


def paper_speedup_kv_only_gdn(d, m, L):
    """Exact GDN form."""
    return (4 * d * d + Fraction(8 * d * d, m) + 2 * m * d + 14 * d + m + 7) / Fraction(4 * L * d + 8 * d + 2 * L + 4)


def paper_optimal_chunk(d):
    """Integer argmax of Eq. 6 over m (P:160 says m = 2 sqrt(d))."""
    return max(range(1, 4 * d), key=lambda m: paper_speedup_chunkwise(d, m))


def paper_capacity_ratio(n_draft, record_bytes_per_token=0, d=128):
    """Concurrent-request ratio, buffered vs recurrent verification
    (P:195-198): recurrent keeps 1 + N states, buffered 1 state + N records."""
    st = 4 * d * d
    return Fraction((1 + n_draft) * st, st + n_draft * record_bytes_per_token)


# ----------------------------------------------------------------- this build


@dataclass(frozen=True)
class LayerBytes:
    """Per slot-layer byte sizes (Appendix B of SURVEY.md)."""
    st: int      # fp32 state, all V heads
    inp: int     # q, k (QK heads), v (V heads) in in_dtype + alpha, beta fp32
    rec: int     # one buffered record: k (QK heads) + u (V heads) + G
    o: int       # fp32 outputs

    @classmethod
    def make(cls, Hk=16, Hv=32, d=128, in_bytes=2, u_bytes=4, keep_raw=False):
        st = 4 * Hv * d * d
        inp = 2 * Hk * d * in_bytes + Hv * d * in_bytes + 8 * Hv
        rec = Hk * d * in_bytes + Hv * d * u_bytes + 4 * Hv
        if keep_raw:
            rec += Hv * d * in_bytes + 4 * Hv
        return cls(st, inp, rec, 4 * Hv * d)

    # one call, one slot
    def decode(self, j):
        """Buffered decode at occupancy j: read S + inputs + j records,
        write o + the new record."""
        return self.st + self.inp + j * self.rec + self.o + self.rec

    def flush(self, n):
        """Fold of n records: read S + n records, write S."""
        return 2 * self.st + n * self.rec if n > 0 else 0

    def cycle_avg(self, C):
        """Average bytes per token over a full buffer cycle (C decodes + 1 flush)."""
        return Fraction(sum(self.decode(j) for j in range(C)) + self.flush(C), C)

    def recurrent(self):
        """Kernel (5a): read S + inputs, write S + o."""
        return 2 * self.st + self.inp + self.o

    def verify(self, N, j0=0):
        return self.st + N * self.inp + j0 * self.rec + N * self.o + N * self.rec

    def commit(self, j0, n_acc):
        n = j0 + n_acc
        return 2 * self.st + n * self.rec if n > 0 else 0

    def recurrent_verify(self, N):
        return self.st + N * self.inp + N * self.st + N * self.o

    def recurrent_commit(self, n_acc):
        return 2 * self.st if n_acc > 0 else 0

    def direct(self, L, n_new=1):
        """Direct decode of n_new tokens at context L (records read once)."""
        return L * self.rec + n_new * (self.inp + self.o + self.rec)
