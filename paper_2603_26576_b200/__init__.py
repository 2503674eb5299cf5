"""B200-native engine for the heteff hot path: state-interval traces -> the
host + device POP/TALP efficiency trees (arXiv 2603.26576).

Drop-in for the reference package's hot-path API (``heteff/__init__.py:3-51``):
the trace model types plus ``validate``, ``summarize_host``,
``summarize_device``, ``host_metrics``, ``device_metrics`` and
``compute_report``, all computed by hand-written sm_100a CUDA kernels behind
the C ABI in ``include/heteff_b200.h``.  Large traces use the columnar path
(:mod:`.engine` ``analyze_device``) with the SoA already in HBM.
"""

from .api import (
    AnalysisError,
    DeviceMetrics,
    DeviceSummary,
    HostMetrics,
    HostSummary,
    MetricsReport,
    RegionReport,
    compute_report,
    device_metrics,
    host_metrics,
    region_reports,
    summarize_device,
    summarize_host,
    validate,
)
from .intervals import EMPTY, FlatSet, complement, flatten, intersect, subtract, total_duration
from .model import (
    U64_MAX,
    DeviceActivityKind,
    DeviceDecl,
    DeviceRecord,
    HostRecord,
    HostState,
    Interval,
    InvalidTraceError,
    Trace,
    ValidationReport,
)
from .report import RenderOptions, render_json, render_text
from .trace_io import (
    CategoryMapping,
    MappingError,
    MappingRule,
    TraceFormatError,
    import_mapped,
    import_mapped_packed,
    read_mapping,
    read_trace,
    read_trace_packed,
    write_trace,
)

__version__ = "0.1.0"

__all__ = [
    "EMPTY", "FlatSet", "complement", "flatten", "intersect", "subtract", "total_duration",
    "AnalysisError", "DeviceMetrics", "DeviceSummary", "HostMetrics", "HostSummary", "MetricsReport",
    "RegionReport", "region_reports", "compute_report", "device_metrics", "host_metrics", "summarize_device", "summarize_host", "validate",
    "U64_MAX", "DeviceActivityKind", "DeviceDecl", "DeviceRecord", "HostRecord", "HostState", "Interval",
    "InvalidTraceError", "Trace", "ValidationReport",
    "RenderOptions", "render_json", "render_text",
    "CategoryMapping", "MappingError", "MappingRule", "TraceFormatError", "import_mapped", "import_mapped_packed",
    "read_mapping", "read_trace", "read_trace_packed", "write_trace",
]
