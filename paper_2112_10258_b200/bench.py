"""volkey.bench drop-in name: the stage-timing harness lives in timing.py."""

from .timing import (DEFAULT_SWEEP_CHUNKS, STAGES, DeviceStageRecorder, StageRecorder, StageTiming, SweepResult,  # noqa: F401
                     TimingSummary, chunk_sweep, emit_csv, read_csv, time_pipeline)
