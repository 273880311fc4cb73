"""Error hierarchy of the reference (strandkit/errors.py:4-25).

When the reference package is importable the drop-in raises the reference's
own classes (so ``except strandkit.errors.DataError`` keeps working after
``install()``); otherwise identical standalone mirrors are used.
"""

try:  # pragma: no cover - depends on the host environment
    from strandkit.errors import (  # type: ignore
        ConfigError,
        DataError,
        PipelineError,
        StrandkitError,
    )
except Exception:  # noqa: BLE001
    class StrandkitError(Exception):
        """Base class for all toolkit errors."""

    class ConfigError(StrandkitError):
        """Invalid configuration value or unknown configuration key."""

    class DataError(StrandkitError):
        """Malformed or missing input data (files, bundles, clouds)."""

    class PipelineError(StrandkitError):
        """A pipeline stage produced an unusable result (e.g. empty output)."""

__all__ = ["StrandkitError", "ConfigError", "DataError", "PipelineError"]
