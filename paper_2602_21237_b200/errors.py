"""Exception classes of the B200 tensor path.

Mirrors the reference hierarchy (/root/reference/pkg/src/relab/errors.py:10-43)
so callers catch the same names. When the drop-in is installed into a live
``relab`` package (``paper_2602_21237_b200.patch``), the operators raise
relab's own classes instead (see ``bind_reference_types``).
"""

from __future__ import annotations


class RelabError(Exception):
    """Root of every error the tensor path diagnoses itself."""


class UnknownAttribute(RelabError):
    """Attribute missing from a schema, or of a type the operator cannot use."""


class OutputTooLarge(RelabError):
    """A join would produce more rows than the caller's cap (raised before
    any output is allocated, tensorpath.py:151-152)."""


class DigestMismatch(RelabError):
    """Repeated runs of one experiment disagreed on their result digest."""


class EmptySamples(RelabError):
    """A percentile was requested over no samples."""


class DeviceError(RelabError, RuntimeError):
    """The CUDA library reported a failure (CUDA error, workspace misuse)."""
