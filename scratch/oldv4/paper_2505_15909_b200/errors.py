"""Exception classes mirroring proj/core/include/rtnq/error.hpp, keyed by the
C-ABI status codes of include/rtnq_capi.h."""


class Error(RuntimeError):
    """rtnq::Error (error.hpp:12-17)."""


class InvalidInputError(Error):
    """rtnq::InvalidInputError (error.hpp:19-23)."""


class ShapeError(Error):
    """rtnq::ShapeError (error.hpp:25-29)."""


class CorruptDataError(Error):
    """rtnq::CorruptDataError (error.hpp:31-35)."""


class PlanError(Error):
    """rtnq::PlanError (error.hpp:37-53); ``offset`` is the byte offset or None."""

    def __init__(self, msg, offset=None):
        super().__init__(msg)
        self.offset = offset


class IoError(Error):
    """rtnq::IoError (error.hpp:55-59)."""


class CudaError(Error):
    """No usable CUDA device, or a launch failed (no reference analogue)."""


class UnsupportedError(Error):
    """The chosen kernel cannot run this shape/dtype combination."""


_BY_STATUS = {1: InvalidInputError, 2: ShapeError, 3: CorruptDataError, 4: PlanError,
              5: IoError, 6: CudaError, 7: Error, 8: UnsupportedError}


def raise_for(status: int, msg: str):
    raise _BY_STATUS.get(status, Error)(msg)
