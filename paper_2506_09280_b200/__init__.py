"""B200-native tensor-comparison hot path of the TTrace silent-bug detector.

Drop-in for the compare path of the reference package `traindiff`
(pkg/src/traindiff/__init__.py:7-36): the same names for trace records,
shard canonicalisation, the perturbation tolerance estimator and the
per-id verdicts, with the arithmetic in hand-written sm_100a kernels behind
the C ABI in include/td_api.h (libtdb200.so).  No CPU fallback: without the
library or a GPU the numeric entry points raise.
"""

from .canonical import (CanonicalId, ReplicaGroup, ShardMapping, SliceBox, TensorKind,
                        canonical_layer_index, check_replicas, identity_mapping, locate_layer,
                        merge, parse_canonical, validate_mapping, whole_box)
from .checker import (CheckEntry, CheckPlan, CheckReport, StaticReport, ToleranceMap, check,
                      check_streaming, compare_static, estimate_tolerance, estimate_tolerance_streaming,
                      render_report)
from .errors import (ConfigInvalid, DigestMismatch, FormatError, MappingInvalid, MergeConflict,
                     NonFinite, ReplicaMismatch, ShapeMismatch, TraindiffError, UnknownBugId)
from .generation import (GenSpec, Normal, SplitMix64, TokenIds, Uniform, extract_shard, fnv1a_64,
                         generate_full, seed_from, signed_uniforms)
from .perturb import PerturbSpec, apply_perturbation
from .tensor import (POLICIES, FloatFormat, PrecisionPolicy, Tensor, frobenius_norm, quantize,
                     quantize_array, rel_err, rel_err_arrays)
from .tracestore import (RankMeta, Trace, TraceCollector, TraceFilter, TraceRecord, pack_pinned,
                         read_trace, trace_from_bytes, trace_to_bytes, write_trace)

__version__ = "0.1.0"
