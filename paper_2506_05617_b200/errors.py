"""Exception taxonomy of the drop-in API.

Names and base class match the reference package (pkg/src/convspectra/
errors.py:4-70) so callers' ``except`` clauses keep working; only the
classes the LFA path can raise carry behaviour.
"""


class ConvSpectraError(Exception):
    """Root of every error this package raises (errors.py:4)."""


class NonFiniteWeight(ConvSpectraError):
    """Weight tensor holds NaN/Inf; ``index`` is the first offending entry."""

    def __init__(self, index, value):
        self.index = tuple(int(i) for i in index)
        self.value = value
        super().__init__(f"non-finite weight {value!r} at index {self.index}")


class ZeroDimension(ConvSpectraError):
    """Some channel count, kernel extent or torus side is smaller than 1."""


class AllocationFailure(ConvSpectraError):
    """The symbol field (or a device buffer) would not fit its memory budget."""


class ConvergenceFailure(ConvSpectraError):
    """Jacobi reached max_sweeps (or met NaN/Inf) on some frequency block."""


class IndexOutOfRange(ConvSpectraError):
    """Requested singular-vector column does not exist."""


class ShapeMismatch(ConvSpectraError):
    """A field or vector does not have the shape the operation expects."""


# Raised only by reference subsystems that are out of scope here (explicit
# matrix, NPY reader, analysis, bench fits); defined so imports resolve.
class KernelLargerThanTorus(ConvSpectraError):
    pass


class SizeCapExceeded(ConvSpectraError):
    pass


class EmptySpectrum(ConvSpectraError):
    pass


class InsufficientPoints(ConvSpectraError):
    pass


class BadMagic(ConvSpectraError):
    pass


class UnsupportedDescr(ConvSpectraError):
    pass


class FortranOrderUnsupported(ConvSpectraError):
    pass


class ShapeRankNot4(ConvSpectraError):
    pass


class TruncatedPayload(ConvSpectraError):
    pass
