"""Exception hierarchy of the tokenizer API.

Same class names and base (TokenizerError) as the reference
(/root/reference/pkg/src/lanebpe/errors.py:8-69) so callers that catch the
reference's exceptions keep working.  DeviceError is new: it carries failures
of the CUDA engine (launch errors, out of memory, missing extension).
"""

from __future__ import annotations


class TokenizerError(Exception):
    """Root of every error raised by this package."""


def _leaf(name: str, doc: str) -> type:
    return type(name, (TokenizerError,), {"__doc__": doc, "__module__": __name__})


MalformedVocab = _leaf("MalformedVocab", "Vocabulary is not a JSON object of symbol -> integer id.")
MissingSymbol = _leaf("MissingSymbol", "Some byte value has no single-symbol id in the vocabulary.")
UnknownTokenId = _leaf("UnknownTokenId", "Token id is unknown or does not map back to bytes.")
MalformedLine = _leaf("MalformedLine", "A merges line is not exactly two space-separated symbols.")
UnknownSymbol = _leaf("UnknownSymbol", "A merges line names a symbol the vocabulary lacks.")
DuplicatePair = _leaf("DuplicatePair", "Two merge rules share the same (left, right) pair.")
ReservedKey = _leaf("ReservedKey", "A pair packs to the key reserved for empty table slots.")
OutOfRange = _leaf("OutOfRange", "Merge position does not address an adjacent pair.")
SequenceTooLong = _leaf("SequenceTooLong", "Input exceeds the configured maximum sequence length.")
InvalidBudget = _leaf("InvalidBudget", "Chunk budget too small to hold a mergeable pair.")
CorpusTooSmall = _leaf("CorpusTooSmall", "Benchmark corpus cannot supply the requested window.")
EmptyRecords = _leaf("EmptyRecords", "Report requested over zero benchmark records.")
MalformedGoldenFile = _leaf("MalformedGoldenFile", "Golden token file has an unknown layout.")
DeviceError = _leaf("DeviceError", "The CUDA engine failed (launch, memory, or missing extension).")


class BatchError(TokenizerError):
    """One input of a batch failed; `input_index` says which."""

    def __init__(self, input_index: int, message: str):
        super().__init__(f"input {input_index}: {message}")
        self.input_index = input_index
