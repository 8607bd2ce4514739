"""Spin strings, determinants, selected bases and sample ingestion (host side).

A configuration is a pair of 64-bit occupation masks ("half-bitstrings"),
bit p set when spatial orbital p is occupied.  The packed view puts alpha in
the low ``norb`` bits (reference ``basis.py:39-47``).  In product mode the
determinant (ia, ib) has the global index ``ia * n_beta + ib`` with strings
kept in *caller* order (reference ``basis.py:208-213``) -- the device tables
and the sigma build index x and sigma exactly this way.

The excitation helpers here (``single_phase``, ``enumerate_singles``,
``enumerate_doubles``) are the small host-side API the reference exports
(``basis.py:62-103``); the production table build runs on the GPU
(:func:`paper_2601_16637_b200.tables.build_excitation_table`).
"""

from __future__ import annotations

from collections import Counter
from dataclasses import dataclass, field
from itertools import combinations
from typing import Iterable, NamedTuple, Union

import numpy as np

__all__ = [
    "SpinString",
    "Determinant",
    "SampleFormatError",
    "IngestReport",
    "SelectedBasis",
    "ExcitationTable",
    "popcount",
    "single_phase",
    "enumerate_singles",
    "enumerate_doubles",
    "ingest_samples",
    "parse_sample_lines",
    "det_to_line",
]

SpinString = int


class Determinant(NamedTuple):
    alpha: SpinString
    beta: SpinString

    def packed(self, norb: int) -> int:
        return self.alpha | (self.beta << norb)


class SampleFormatError(ValueError):
    def __init__(self, message: str, line_no: int):
        super().__init__(f"line {line_no}: {message}")
        self.line_no = line_no


def popcount(s: int) -> int:
    return int(s).bit_count()


def _between_mask(p: int, r: int) -> int:
    lo, hi = min(p, r), max(p, r)
    return ((1 << hi) - 1) ^ ((1 << (lo + 1)) - 1)


def single_phase(s: SpinString, p: int, r: int) -> int:
    """(-1)^(occupied orbitals strictly between p and r) -- reference basis.py:62-69."""
    return -1 if popcount(s & _between_mask(p, r)) & 1 else 1


def _occ_virt(s: int, norb: int):
    occ = [o for o in range(norb) if s >> o & 1]
    return occ, [o for o in range(norb) if not s >> o & 1]


def enumerate_singles(s: SpinString, norb: int):
    """(target, p, r, phase) for p occupied ascending, r virtual ascending."""
    occ, virt = _occ_virt(s, norb)
    return [((s ^ (1 << p)) | (1 << r), p, r, single_phase(s, p, r)) for p in occ for r in virt]


def enumerate_doubles(s: SpinString, norb: int):
    """(target, p, q, r, s, phase): lexicographic (p<q) x (r<s), sequential-single phase."""
    occ, virt = _occ_virt(s, norb)
    out = []
    for p, q in combinations(occ, 2):
        for r, t in combinations(virt, 2):
            mid = (s ^ (1 << p)) | (1 << r)
            out.append(((mid ^ (1 << q)) | (1 << t), p, q, r, t,
                        single_phase(s, p, r) * single_phase(mid, q, t)))
    return out


@dataclass(frozen=True)
class IngestReport:
    n_lines: int
    n_filtered: int
    n_duplicates: int
    det_counts: Counter = field(default_factory=Counter)


@dataclass
class SelectedBasis:
    """Product (alpha x beta) or explicit determinant subspace (reference basis.py:118-223)."""

    mode: str
    norb: int
    n_alpha_elec: int
    n_beta_elec: int
    alpha_strings: list = field(default_factory=list)
    beta_strings: list = field(default_factory=list)
    dets: list = field(default_factory=list)
    _alpha_index: dict = field(default_factory=dict, repr=False)
    _beta_index: dict = field(default_factory=dict, repr=False)
    _det_index: dict = field(default_factory=dict, repr=False)

    @staticmethod
    def _validate(strings, norb, n_elec, label):
        for s in strings:
            if s < 0 or s >> norb:
                raise ValueError(f"{label} string {s:#x} has bits above orbital {norb - 1}")
            if popcount(s) != n_elec:
                raise ValueError(f"{label} string {s:#x} has {popcount(s)} electrons, expected {n_elec}")

    @classmethod
    def product(cls, alpha_strings: Iterable[int], beta_strings: Iterable[int],
                norb: int, n_alpha_elec: int, n_beta_elec: int) -> "SelectedBasis":
        alphas = [int(s) for s in alpha_strings]
        betas = [int(s) for s in beta_strings]
        cls._validate(alphas, norb, n_alpha_elec, "alpha")
        cls._validate(betas, norb, n_beta_elec, "beta")
        return cls("product", norb, n_alpha_elec, n_beta_elec, alphas, betas,
                   _alpha_index={s: i for i, s in enumerate(alphas)},
                   _beta_index={s: i for i, s in enumerate(betas)})

    @classmethod
    def explicit(cls, dets: Iterable, norb: int, n_alpha_elec: int, n_beta_elec: int) -> "SelectedBasis":
        dl = [Determinant(int(d[0]), int(d[1])) for d in dets]
        cls._validate([d.alpha for d in dl], norb, n_alpha_elec, "alpha")
        cls._validate([d.beta for d in dl], norb, n_beta_elec, "beta")
        index = {d: i for i, d in enumerate(dl)}
        if len(index) != len(dl):
            raise ValueError("duplicate determinants in explicit basis")
        return cls("explicit", norb, n_alpha_elec, n_beta_elec, dets=dl, _det_index=index)

    @property
    def dimension(self) -> int:
        if self.mode == "product":
            return len(self.alpha_strings) * len(self.beta_strings)
        return len(self.dets)

    def alpha_index(self, s: int) -> int:
        return self._alpha_index[s]

    def beta_index(self, s: int) -> int:
        return self._beta_index[s]

    def index_of(self, det) -> int:
        if self.mode == "product":
            return self._alpha_index[det[0]] * len(self.beta_strings) + self._beta_index[det[1]]
        return self._det_index[Determinant(*det)]

    def det_at(self, i: int) -> Determinant:
        if not 0 <= i < self.dimension:
            raise IndexError(f"index {i} out of range [0, {self.dimension})")
        if self.mode == "product":
            ia, ib = divmod(i, len(self.beta_strings))
            return Determinant(self.alpha_strings[ia], self.beta_strings[ib])
        return self.dets[i]

    # device-facing views
    def alpha_array(self) -> np.ndarray:
        return np.asarray(self.alpha_strings, dtype=np.uint64)

    def beta_array(self) -> np.ndarray:
        return np.asarray(self.beta_strings, dtype=np.uint64)


def det_to_line(det: Determinant, norb: int) -> str:
    bits = lambda w: "".join("1" if w >> p & 1 else "0" for p in range(norb))  # noqa: E731
    return bits(det.alpha) + bits(det.beta)


def _parse_line(line: str, norb: int, line_no: int) -> Determinant:
    if len(line) != 2 * norb:
        raise SampleFormatError(f"expected {2 * norb} characters, got {len(line)}", line_no)
    bad = set(line) - {"0", "1"}
    if bad:
        ch = next(c for c in line if c in bad)
        raise SampleFormatError(f"character {ch!r} is not '0' or '1'", line_no)
    a = sum(1 << p for p, c in enumerate(line[:norb]) if c == "1")
    b = sum(1 << p for p, c in enumerate(line[norb:]) if c == "1")
    return Determinant(a, b)


def parse_sample_lines(lines: Union[str, Iterable[str]], norb: int):
    """Sampled 0/1 text lines -> (alpha uint64[n], beta uint64[n]) in file order (host text layer).

    Reference line format (``basis.py:231-248``): 2*norb characters, leftmost =
    orbital 0 of alpha; blank lines and '#' comments skipped; the first
    malformed line raises SampleFormatError with its 1-based line number.
    """
    if not 1 <= norb <= 64:
        raise ValueError(f"sample ingestion takes norb in [1, 64] (one-word strings), got {norb}")
    if isinstance(lines, str):
        lines = lines.splitlines()
    kept, nos = [], []
    for line_no, raw in enumerate(lines, start=1):
        line = raw.strip()
        if not line or line[0] == "#":
            continue
        kept.append(line)
        nos.append(line_no)
    n = len(kept)
    if n == 0:
        return np.zeros(0, np.uint64), np.zeros(0, np.uint64)
    w = 2 * norb
    lens = np.fromiter(map(len, kept), dtype=np.int64, count=n)
    text = "".join(kept)
    ascii_ok = text.isascii()
    if ascii_ok and (lens == w).all():
        chars = np.frombuffer(text.encode("ascii"), dtype=np.uint8).reshape(n, w)
        bad_rows = np.nonzero(((chars != 48) & (chars != 49)).any(axis=1))[0]
        first_bad = int(bad_rows[0]) if bad_rows.size else n
    else:
        first_bad = 0  # locate the first malformed line the slow way below
    if first_bad < n:
        for line, line_no in zip(kept[first_bad:], nos[first_bad:]):
            _parse_line(line, norb, line_no)  # raises at the first malformed line, reference order
    bits = chars == 49
    weights = np.zeros((n, 64), dtype=bool)

    def pack(block):
        weights[:, :norb] = block
        return np.packbits(weights, axis=1, bitorder="little").view(np.uint64).reshape(n)

    return pack(bits[:, :norb]).copy(), pack(bits[:, norb:]).copy()


def ingest_samples(lines: Union[str, Iterable[str]], norb: int, n_alpha_elec: int,
                   n_beta_elec: int, mode: str = "product", device=None):
    """Sampled 0/1 lines -> (SelectedBasis, IngestReport); first-seen order kept.

    Contract of reference ``basis.py:251-313``: leftmost character is orbital
    0 of alpha; blank and '#' lines skipped; wrong popcounts filtered;
    duplicates dropped; product mode spans unique alpha x unique beta halves.
    The text is parsed on the host (``parse_sample_lines``); filtering,
    deduplication, multiplicities and the unique halves run on the GPU
    (``sbd_ingest_samples`` via ``ingest_sample_arrays``).
    """
    from .ingest import ingest_sample_arrays

    mode = mode.lower()
    if mode not in ("product", "explicit"):
        raise ValueError(f"mode must be 'product' or 'explicit', got {mode!r}")
    a, b = parse_sample_lines(lines, norb)
    return ingest_sample_arrays(a, b, norb, n_alpha_elec, n_beta_elec, mode=mode, device=device)


@dataclass
class ExcitationTable:
    """CSR in-set excitations of one spin sector (reference ``basis.py:316-359``).

    Row i = source string i (caller order); entries in enumeration order;
    targets are caller-order indices.  Built on the device.
    """

    n_strings: int
    norb: int
    s_off: np.ndarray
    s_tgt: np.ndarray
    s_hole: np.ndarray
    s_part: np.ndarray
    s_phase: np.ndarray
    d_off: np.ndarray
    d_tgt: np.ndarray
    d_hole1: np.ndarray
    d_hole2: np.ndarray
    d_part1: np.ndarray
    d_part2: np.ndarray
    d_phase: np.ndarray

    def singles_of(self, i: int):
        lo, hi = int(self.s_off[i]), int(self.s_off[i + 1])
        return [(int(self.s_tgt[k]), int(self.s_hole[k]), int(self.s_part[k]), int(self.s_phase[k]))
                for k in range(lo, hi)]

    def doubles_of(self, i: int):
        lo, hi = int(self.d_off[i]), int(self.d_off[i + 1])
        return [(int(self.d_tgt[k]), int(self.d_hole1[k]), int(self.d_hole2[k]),
                 int(self.d_part1[k]), int(self.d_part2[k]), int(self.d_phase[k]))
                for k in range(lo, hi)]

    @property
    def mean_connections(self) -> float:
        """c-bar: in-set singles + doubles per string (roofline input)."""
        n = max(self.n_strings, 1)
        return float(self.s_off[-1] + self.d_off[-1]) / n
