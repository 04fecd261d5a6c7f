"""B200-native Astra Mixed-Precision Attention inference (arXiv 2505.19342).

Drop-in for the inference surface of the reference package ``seqvq`` (its package-level
names for the hot path, seqvq/__init__.py): the operator API (VQ, attention), the
sequence-parallel runtime (``run_inference``), the model API, the codebook setup, the
communication model and the error taxonomy, all over the native sm_100a library
(``_lib/libastra_b200.so``, C ABI in ``include/astra_b200.h``).  Training, the theorem lab and
the config/CLI layer of the reference are out of scope.
"""

from .attention import (MixedPrecisionMask, build_mask, mixed_precision_attention,
                        multihead_attention, softmax_perturbation_first_order,
                        standard_attention)
from .cluster import (LEDGER_COLUMNS, CommsLedger, InferenceResult, ShardPlan,
                      partition_tokens, run_inference)
from .codebooks import fit_codebooks, initialize_codebooks, kmeans_init
from .comms import (BENCH_COLUMNS, METHODS, CommsConfig, LinkModel, MethodSpec, astra_wire_bytes,
                    bench_csv, comm_time, compute_time, fit_link, measure_allgather,
                    speedup_table_measured)
from .data import make_classify_data
from .errors import (ConfigError, IndexCorruptionError, LifecycleError, MaskError, ModeError,
                     PlanError, ProtocolError, ShapeError)
from .model import (DecodeState, ModelConfig, ModelParams, Tensor, aggregate_class_tokens,
                    classify, embed_classifier_inputs, embed_lm_inputs,
                    exact_codebooks_from_reference, generate, generator, init_params,
                    lm_logits, load_checkpoint, prefill_decode_state, run_blocks,
                    save_checkpoint)
from .vq import (Codebook, QuantizedTokens, dequantize, index_bits, load_codebook, quantize,
                 save_codebook)

__version__ = "0.2.0"
