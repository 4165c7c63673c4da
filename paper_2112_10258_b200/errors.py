"""Error taxonomy of the drop-in API (mirrors volkey errors.py:8-53).

Native status codes from ``libvolkey_b200`` map onto these classes in
``_lib.check``: 5 -> ParameterError, 7 -> DataError; CUDA failures raise
``DeviceError`` (not a reference class: the reference has no device).
"""


class VolkeyError(Exception):
    kind = "error"
    exit_code = 1


class InputOutputError(VolkeyError):
    kind = "io"
    exit_code = 3


class FormatError(VolkeyError):
    kind = "format"
    exit_code = 4


class ParameterError(VolkeyError):
    kind = "parameter"
    exit_code = 5


class NoConsensusError(VolkeyError):
    kind = "no_consensus"
    exit_code = 6


class DataError(VolkeyError):
    kind = "data"
    exit_code = 7


class DeviceError(VolkeyError):
    """CUDA launch/runtime failure or missing GPU/extension (no CPU fallback)."""

    kind = "device"
    exit_code = 20


EXIT_CODES = {c.kind: c.exit_code for c in (VolkeyError, InputOutputError, FormatError, ParameterError,
                                            NoConsensusError, DataError, DeviceError)}
