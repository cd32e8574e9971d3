"""B200-native (sm_100a) DICM / AMS training hot path.

A drop-in for the reference's training step (arXiv 1711.06505 re-implementation,
package ``dicm``): same model description, parameter names and initial values,
same ``LocalTrainer`` / ``Cluster`` step API, with every op of the step running
in hand-written CUDA kernels behind the C ABI in ``include/dicm_b200.h``.

Importing the package does not need a GPU; constructing a model or a pool does.
"""

from .schema import (AGGREGATOR_KINDS, AggregatorSpec, FeatureSchema, FieldSpec, ModelLayout,  # noqa: F401
                     TowerSpec, default_schema, image_net_widths, init_params, param_specs)
from .batch import Batch, encode_batch, synthetic_batch  # noqa: F401

__all__ = ["AGGREGATOR_KINDS", "AggregatorSpec", "FeatureSchema", "FieldSpec", "ModelLayout", "default_schema",
           "image_net_widths", "init_params", "param_specs", "Batch", "encode_batch", "synthetic_batch",
           "DicmModel", "ImagePool", "FixedExtractor", "LocalTrainer", "TrainConfig", "StepEngine", "Cluster",
           "ClusterConfig", "run_training", "InferenceTable", "KvPredictor", "export_inference",
           "predict_logits", "checkpoint", "PrerankModel", "forward_ctr", "forward_prerank", "TowerSpec"]


def __getattr__(name):
    # device-side classes load the kernel library lazily (ImportError if missing)
    if name in ("DicmModel", "PrerankModel"):
        from . import model
        return getattr(model, name)
    if name in ("ImagePool", "FixedExtractor"):
        from . import pool
        return getattr(pool, name)
    if name in ("LocalTrainer", "TrainConfig", "TrainLog", "minibatches"):
        from . import training
        return getattr(training, name)
    if name == "StepEngine":
        from .engine import StepEngine
        return StepEngine
    if name in ("InferenceTable", "KvPredictor", "export_inference", "predict_logits", "forward_ctr",
                "forward_prerank"):
        from . import inference
        return getattr(inference, name)
    if name in ("Cluster", "ClusterConfig", "run_training"):
        from . import runtime
        return getattr(runtime, name)
    raise AttributeError(name)
