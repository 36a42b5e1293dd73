"""paper_2605_25521_b200 -- B200-native PQ construction (encode + Lloyd codebook
training), a drop-in for the hot path of the reference package ``cspq``
(/root/reference/pkg/src/cspq/__init__.py:9-100).

The compute runs in hand-written sm_100a CUDA kernels behind the C ABI of
include/cspq_b200.h (library: _lib/libcspq_b200.so); this package is the
host-side mirror of the reference's API: same names, argument meanings,
layouts and exceptions.  There is no CPU fallback.
"""

from .core import (
    Codebook,
    ConfigError,
    CorruptionError,
    DataError,
    Error,
    FormatError,
    PQCodes,
    PQParams,
    ScoreBlock,
    TrainingError,
    VectorDataset,
    compute_biases,
    partition_vector,
    transpose_codebook,
)
from .kernels import (
    EncoderVariant,
    encode_blocked,
    encode_blocked_with_score,
    encode_ref,
    encode_ref_with_score,
    encode_reform,
    encode_reform_with_score,
    encode_vector,
    native_lane_width,
)
from .training import (
    KMeansResult,
    TrainConfig,
    lloyd_iterate,
    lloyd_iterate_batched,
    run_lloyd,
    train_all_codebooks,
    train_all_codebooks_report,
    train_codebook,
    train_codebook_report,
)
from .bulk import (
    CHUNK_MAJOR,
    VECTOR_MAJOR,
    CodebookSet,
    ExecutionPlan,
    encode_dataset,
    encode_dataset_device,
    encode_dataset_host,
    estimate_working_set,
)
from .io import (
    crc32_device,
    encode_file,
    read_bvecs,
    read_codebooks,
    read_codes,
    read_fvecs,
    read_ivecs,
    synth_dataset,
    write_bvecs,
    write_codebooks,
    write_codes,
    write_fvecs,
    write_ivecs,
)
from .evaluation import EvalReport, adc_search, adc_search_batched, evaluate, exact_topn, mse_of, reconstruct
from ._device import pinned_empty
from ._native import NativeUnavailable

__version__ = "0.1.0"

from .harness import BENCH_CSV_COLUMNS, BenchResult, run_bench_matrix, run_verify, write_bench_csv  # noqa: E402

__all__ = [
    "BENCH_CSV_COLUMNS", "BenchResult", "run_bench_matrix", "run_verify", "write_bench_csv",
    "EvalReport", "adc_search", "adc_search_batched", "evaluate", "exact_topn", "mse_of", "reconstruct",
    "crc32_device", "encode_file", "read_bvecs", "read_codebooks", "read_codes", "read_fvecs", "read_ivecs",
    "synth_dataset", "write_bvecs", "write_codebooks", "write_codes", "write_fvecs", "write_ivecs",
    "CHUNK_MAJOR", "VECTOR_MAJOR", "Codebook", "CodebookSet", "ConfigError", "CorruptionError",
    "DataError", "EncoderVariant", "Error", "ExecutionPlan", "FormatError", "KMeansResult",
    "NativeUnavailable", "PQCodes", "PQParams", "ScoreBlock", "TrainConfig", "TrainingError",
    "VectorDataset", "compute_biases", "encode_blocked", "encode_blocked_with_score",
    "encode_dataset", "encode_dataset_device", "encode_dataset_host", "encode_ref",
    "encode_ref_with_score", "encode_reform", "encode_reform_with_score", "encode_vector",
    "estimate_working_set", "lloyd_iterate", "lloyd_iterate_batched", "native_lane_width",
    "partition_vector", "pinned_empty", "run_lloyd", "train_all_codebooks",
    "train_all_codebooks_report", "train_codebook", "train_codebook_report",
    "transpose_codebook", "__version__",
]
