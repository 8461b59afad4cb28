"""Alias of ``harness`` under the reference's module name (``moaprod.bench``),
so ``from <package>.bench import run_experiment`` keeps working."""

from .harness import (METRIC_FIELDS, MODES, RAW_FIELDS, ExperimentConfig,  # noqa: F401
                      ExperimentResult, MetricRow, SizeFailure, TimingRecord, derive_metrics,
                      emit_csv, operand_pair, read_records_csv, run_experiment)
