"""B200-native GPT-2 byte-level BPE encoder.

Drop-in for the encode path of the reference package `lanebpe`
(/root/reference/pkg): same construction API (Vocab / parse_merges /
build_table / Tokenizer / BlockConfig), same batch API (tokenize_batch ->
BatchResult, TokenizerHandle.tokenize_batch), same exceptions -- with the
merge loop running as hand-written sm_100a CUDA kernels behind the C ABI in
include/gpubpe.h (libgpubpe.so, built in-tree).  No CPU fallback.
"""

from . import errors
from .bindings import TokenizerHandle
from .byte_codec import ByteEncoder, Vocab, base_id_table, build_byte_encoder, decode_tokens, encode_bytes
from .chunker import ENGINE_NAMES, BatchResult, Chunk, Tokenizer, chunk_tokens, pack_texts, tokenize_batch
from .engine import (
    BlockConfig,
    PairCandidate,
    PassCounters,
    compact_double_buffer,
    compact_scan,
    eval_pairs,
    inject_compaction_fault,
    run_block_engine,
    sequential_bpe,
    token_seq,
)
from .windows import DEFAULT_LENGTHS, SweepSpec, make_windows
from .report import (
    BenchRecord,
    GoldenReport,
    ProfileReport,
    compare_golden,
    emit_report,
    load_golden_file,
    profile_run,
    run_sweep,
)
from .merge_table import (
    MergeRule,
    PackedPairTable,
    ProbeScratch,
    build_table,
    pack_key,
    pack_value,
    parse_merges,
    rule_arrays,
    unpack_value,
)

__version__ = "0.1.0"


def pinned_empty(nbytes: int, device: int = 0):
    """uint8[nbytes] in pinned, device-mapped host memory; batches packed here
    reach the GPU by DMA without a staging copy (see device.pinned_empty)."""
    from .device import pinned_empty as _pinned_empty

    return _pinned_empty(nbytes, device)

__all__ = [
    "BatchResult", "BenchRecord", "GoldenReport", "ProfileReport", "compare_golden", "emit_report",
    "load_golden_file", "profile_run", "run_sweep", "BlockConfig", "DEFAULT_LENGTHS", "SweepSpec", "make_windows", "ByteEncoder", "Chunk", "ENGINE_NAMES", "MergeRule",
    "PackedPairTable", "PassCounters", "Tokenizer", "TokenizerHandle", "Vocab", "base_id_table",
    "build_byte_encoder", "build_table", "chunk_tokens", "decode_tokens", "encode_bytes", "errors",
    "pack_key", "pack_texts", "pack_value", "pinned_empty", "parse_merges", "rule_arrays", "tokenize_batch",
    "unpack_value", "run_block_engine", "sequential_bpe", "token_seq", "__version__",
    "PairCandidate", "ProbeScratch", "compact_double_buffer", "compact_scan", "eval_pairs",
    "inject_compaction_fault",
]
