"""Error types of the drop-in API.

Same names, hierarchy and meaning as the reference's error tree
(/root/reference/pkg/src/ente/exceptions.py:4-80): every error derives from
EnteError; NonFiniteValue carries the 0-based (rep, t) location.  The plain
subclasses are generated from one table so that the mapping is explicit.
"""

from __future__ import annotations


class EnteError(Exception):
    """Base class for every error of the toolbox."""


class NonFiniteValue(EnteError):
    """A NaN/Inf sample at 0-based (rep, t) (data.py:60-74 of the reference)."""

    def __init__(self, rep: int, t: int):
        self.rep = rep
        self.t = t
        super().__init__(f"non-finite value at repetition {rep}, sample {t} (0-based)")


# name -> when it is raised in this package
_PLAIN = {
    "EmptyEnsemble": "ensemble with R == 0 or N == 0",
    "RaggedRepetitions": "repetitions of unequal length / not a 2-D matrix",
    "IndexUnderflow": "an embedding or window reaches before sample 1",
    "ShapeMismatch": "bad chunk / radii / marginal shapes, non-finite chunk values",
    "InsufficientData": "not enough repetitions or anchors",
    "KTooLarge": "k outside [1, n-1]",
    "DomainError": "digamma outside its domain",
    "DegenerateData": "all pooled points identical",
    "InvalidPermutation": "a surrogate permutation that is not a bijection",
    "UnknownMethod": "unknown multiple-comparison method",
    "ParseError": "unparseable input file",
    "GridIncomplete": "incomplete scan grid",
    "MagicMismatch": "wrong binary file magic",
    "IntegrationDiverged": "simulator blew up",
    "UnstableParameters": "unstable simulator parameters",
    "ResultMismatch": "batched and sequential results differ",
    "IoError": "file I/O failure",
}

for _name, _doc in _PLAIN.items():
    globals()[_name] = type(_name, (EnteError,), {"__doc__": _doc, "__module__": __name__})

__all__ = ["EnteError", "NonFiniteValue", *_PLAIN]
