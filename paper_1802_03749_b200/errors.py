"""Error classes of the indirect-loop engine, plus the C-ABI status mapping.

The class names and hierarchy are the ones ``meshplan`` users catch
(reference: pkg/src/meshplan/errors.py:8-29).  The native library returns an
integer status instead of raising; :func:`raise_for_status` turns a status and
the library's thread-local message into the same exception class, so callers
cannot tell whether a fault was detected on the host or on the device.

Status codes follow the reference CLI exit codes (cli.py:368-377): 2 for
validation / kernel-contract problems, 3 for races, 4 for capacity faults,
5 for file-format problems.  Status 1 is a CUDA runtime failure.
"""


class MeshplanError(Exception):
    """Root of every error raised by this package."""


class MeshValidationError(MeshplanError):
    """The mesh, a configuration knob or a flag combination is invalid."""


class KernelSpecError(MeshplanError):
    """A kernel signature is malformed or has no device implementation."""


class RaceError(MeshplanError):
    """Two parallel writers of one colour group would touch the same point."""


class CapacityError(MeshplanError):
    """A plan needs more than a hardware limit allows (shared bytes, widths)."""


class FileFormatError(MeshplanError):
    """A plan / permutation / partition file cannot be parsed."""


class DeviceError(MeshplanError):
    """The CUDA runtime reported a failure inside the native library."""


# native status -> exception class (include/meshplan_b200.h, MP_STATUS_*)
STATUS_CLASSES = {
    1: DeviceError,
    2: KernelSpecError,
    3: RaceError,
    4: CapacityError,
    5: FileFormatError,
    6: MeshValidationError,
}


def raise_for_status(status: int, message: str) -> None:
    """Raise the exception class registered for a non-zero native status."""
    if status == 0:
        return
    cls = STATUS_CLASSES.get(int(status), MeshplanError)
    raise cls(message or f"native call failed with status {status}")
