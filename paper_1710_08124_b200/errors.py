"""Error types of the drop-in boundary.

Mirrors the reference convention (`pkg/src/fepll/errors.py:8-20`): invalid
inputs raise :class:`DataError`, non-finite results raise
:class:`NumericalError`; CG non-convergence is reported through
``SolveInfo.converged`` and is not an error.  The C-ABI return codes map
onto these classes (0 ok, 3 data error, 4 numerical error, 5 CUDA/launch
failure, which surfaces as :class:`DeviceError`).
"""


class FepllError(Exception):
    """Base class of every error raised by this package."""


class DataError(FepllError):
    """Invalid input: shapes, parameters, model or tree invariants."""


class NumericalError(FepllError):
    """A numerical step produced non-finite values."""


class DeviceError(FepllError):
    """The CUDA library is missing, failed to launch, or reported a fault."""
