"""B200-native KVComp Store/Fetch hot path (arxiv 2509.00579).

Drop-in for the reference package ``kvpack``'s store/fetch/attend API
(kvpack/__init__.py:9-75): the same names and argument meanings, backed by
hand-written sm_100a kernels in ``libkvcomp.so`` (C ABI: include/kvcomp.h).
Tensors live on the CUDA device; results are torch tensors.
"""

from .attention import (AttentionOutput, attention_batched, attention_gqa, attention_step,
                        dense_attention_f16,
                        fused_k_scores, fused_v_output, multistage_attention, reference_output,
                        reference_scores, softmax_rows)
from .codebook import (DecodeTree, HuffmanCodebook, build_codebook, build_histogram,
                       build_smoothed_codebook, codebook_from_lengths, deserialize_codebook,
                       histogram_entropy, serialize_codebook, smooth_histogram)
from .codec import (CompressedArena, CompressedBlock, DataMovement, DeviceArena, compress_block, decode_slice,
                    decode_slices, decompress_block, encode_slice, iter_decoded_blocks, metadata_overhead,
                    reserve_arena_pool, scan_offsets, units_per_block)
from .container import load_state, read_header, save_state
from .errors import (ArenaFullError, CodebookError, CodecError, ConfigError,
                     ContainerFormatError, KvpackError, TensorFormatError)
from .decode_loop import DecodeLoop
from .kvcache import LayerCacheState, append_batched
from .paged import PagedArena, PagePool
from .metrics import (BenchRow, CompressionStats, SimulationResult, SimulationSettings,
                      collect_stats, config_label, equivalent_decompression_throughput,
                      median_time, run_ratio_sweep, run_simulation, write_csv)
from .quantizer import (DEFAULT_REL_SCALE, MIN_REL_SCALE, QuantConfig, QuantizedBlock, QuantMode,
                        QuantUnitMeta, dequantize_block, quantize_block, quantize_unit)
from .tensor_io import (CacheTensor, SyntheticSpec, generate_synthetic, generate_synthetic_device,
                        read_tensor, write_tensor)
from . import bench  # noqa: F401  (kvpack.bench)

__version__ = "0.1.0"
