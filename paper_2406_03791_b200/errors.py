"""Exception taxonomy of the reference (errors.hpp:23-85), raised from the C ABI
status codes of include/rnntg.h (1:1 mapping)."""
import builtins


class Error(RuntimeError):
    """rnntsim::Error"""


class DimensionError(Error):
    """Shape or rank of an operand does not fit the operation."""


class DtypeError(Error):
    """Operand has the wrong element type."""


class IndexError(Error, builtins.IndexError):  # noqa: A001 - mirrors rnntsim::IndexError
    """An index (label id, row, duration class) is out of range."""


class ValueError(Error, builtins.ValueError):  # noqa: A001 - mirrors rnntsim::ValueError
    """A configuration value is outside its documented domain."""


class StateError(Error):
    """Decoder asked to do something inconsistent with its current state."""


class StructureError(Error):
    """A graph violates the structural rules for conditional nodes."""


class RunawayLoopError(Error):
    """A while node exceeded the configured iteration cap."""


class CudaError(Error):
    """CUDA runtime failure or no device (there is no CPU fallback)."""


class AllocError(CudaError):
    """Device allocation failed."""


STATUS = {1: ValueError, 2: DimensionError, 3: DtypeError, 4: IndexError, 5: StateError,
          6: StructureError, 7: RunawayLoopError, 8: CudaError, 9: AllocError}
