"""B200-native Selected Basis Diagonalization (drop-in for the `sbdiag` reference API).

Host side: Python + PyTorch (device memory, streams, torch.distributed/NCCL).
Compute: hand-written sm_100a CUDA kernels in ``libsbd_b200.so`` behind the
C ABI of ``include/sbd.h``.  Public names follow the reference package
(``pkg/src/sbdiag/__init__.py:17-39``).
"""

from __future__ import annotations

from .apply import (
    HamiltonianApplier,
    SpinTables,
    apply_H,
    apply_H_full,
    build_excitation_table,
    build_excitation_table128,
    build_spin_tables,
    compute_diagonal,
    sorted_strings128,
    string_words,
)
from .basis import (
    Determinant,
    ExcitationTable,
    IngestReport,
    SampleFormatError,
    SelectedBasis,
    det_to_line,
    enumerate_doubles,
    enumerate_singles,
    ingest_samples,
    popcount,
    single_phase,
)
from .davidson import DavidsonOptions, DavidsonResult, DavidsonStats, davidson_solve
from .ingest import ingest_sample_arrays, start_vector
from .integrals import FcidumpError, IntegralTable, parse_fcidump, write_fcidump

__all__ = [
    "Determinant",
    "IngestReport",
    "SelectedBasis",
    "ingest_samples",
    "IntegralTable",
    "parse_fcidump",
    "HamiltonianApplier",
    "apply_H",
    "DavidsonOptions",
    "DavidsonResult",
    "davidson_solve",
    # lower-level reference names
    "SpinTables",
    "build_spin_tables",
    "build_excitation_table",
    "compute_diagonal",
    "apply_H_full",
    # B200 extensions: device ingestion
    "ingest_sample_arrays",
    "start_vector",
    # B200 extensions: 128-bit strings (north_star (1)-(2)), tables only
    "build_excitation_table128",
    "sorted_strings128",
    "string_words",
    "ExcitationTable",
    "DavidsonStats",
    "FcidumpError",
    "write_fcidump",
    "SampleFormatError",
    "det_to_line",
    "enumerate_singles",
    "enumerate_doubles",
    "single_phase",
    "popcount",
]

__version__ = "0.1.0"
