"""permlab-b200: a B200-native engine for the Store-zechin permanent
(arXiv 1802.02779), drop-in for the reference's ``permlab::store_zechin_*``
entry points. See DESIGN.md."""
from .api import (  # noqa: F401
    AttributionReport,
    DeviceError,
    DomainError,
    Limits,
    OpCount,
    PermanentResult,
    StoreZechinRun,
    binom,
    colex_rank,
    colex_unrank,
    device_count,
    release_scratch,
    ryser_counts,
    ryser_permanent,
    scratch_bytes,
    store_zechin_attributed,
    store_zechin_counts,
    store_zechin_permanent,
    store_zechin_permanent_batch,
    store_zechin_run,
    version,
)
