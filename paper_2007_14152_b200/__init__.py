"""B200-native sparse-DNN inference (arXiv 2007.14152 hot path), drop-in for ``spdnn``.

The per-layer ``Y <- min(ReLU(Y.W + b), 32)`` loop with dead-feature pruning
runs in hand-written sm_100a CUDA (csrc/layer.cu) behind the C ABI declared
in include/spdnn_b200.h; this package is the host side, mirroring the
reference's Python API (``spdnn/__init__.py:9-63``) name for name.
"""

from .model import (FeatureBatch, InferenceConfig, LayerCSR, ModelError, NetworkModel,
                    count_edges, make_feature_batch, make_layer_csr, relu_clamped,
                    validate_model)
from .ingest import (GeneratorSpec, IngestError, generate_synthetic_inputs,
                     generate_synthetic_network, iter_synthetic_layers, load_features_tsv,
                     load_layer_tsv, load_truth_categories, read_binary, write_binary)
from .engine import (InferenceResult, LayerOutcome, LayerPlan, PaddingStats, PlanParams,
                     PreparedLayer, WeightStreamer, baseline_layer, compact_active, infer,
                     infer_device, optimized_layer,
                     prepare_model, run_layer_step)
from .parallel import (BalanceEntry, BalanceReport, CommMatrix, CountMsg, GatherMsg, Partition,
                       RowsMsg, apply_transfers, balance_step, gather_categories,
                       imbalance_ratio, partition_even, run_batch_parallel)

__version__ = "0.1.0"
