"""``kvpack.bench`` (reference bench.py:1-387) under its own module name, so
``from kvpack.bench import run_simulation`` ports unchanged.  The definitions
live in :mod:`.metrics` (statistics, BenchRow/CSV, the decode-loop simulation
and the ratio sweep, all on the device)."""

from .metrics import (FUSED_FASTER, BenchRow, CompressionStats, SimulationResult, SimulationSettings,  # noqa: F401
                      collect_stats, config_label, equivalent_decompression_throughput,
                      median_time, run_ratio_sweep, run_simulation, write_csv)
# names the reference's bench module also carries (bench.py:25-50 imports)
from .attention import (attention_step, multistage_attention, reference_output,  # noqa: F401,E402
                        reference_scores, softmax_rows)
from .codec import DataMovement  # noqa: F401,E402
from .errors import ConfigError  # noqa: F401,E402
from .kvcache import LayerCacheState  # noqa: F401,E402
from .quantizer import QuantConfig, QuantMode  # noqa: F401,E402
from .tensor_io import CacheTensor, SyntheticSpec, generate_synthetic  # noqa: F401,E402
