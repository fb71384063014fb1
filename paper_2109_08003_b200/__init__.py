"""paper_2109_08003_b200 — B200-native engine for the deep-encoder /
shallow-decoder translation students of NiuTrans' WMT21 efficiency system
(arXiv 2109.08003), drop-in for the reference ``fastnmt`` hot path.

Host-side construction (``ModelConfig``, ``random_model``, ``count_params``)
and scheduling (``batching``) import without a GPU; the model, search and
engine modules load ``libfnmt_b200.so`` and raise if it is missing.
"""

from .store import (BOS_ID, EOS_ID, PAD_ID, UNK_ID, ModelConfig, Weights, count_params,
                    random_model, sinusoid_positions, tensor_manifest)

__version__ = "0.1.0"

__all__ = ["ModelConfig", "Weights", "count_params", "random_model", "sinusoid_positions",
           "tensor_manifest", "PAD_ID", "UNK_ID", "BOS_ID", "EOS_ID", "GpuTranslationModel",
           "Engine", "RunConfig", "Translator", "greedy_translate", "beam_translate", "SearchConfig"]


def __getattr__(name):
    if name in ("GpuTranslationModel", "GpuEncoderOutput", "GpuDecodeCache", "LengthError"):
        from . import model
        return getattr(model, name)
    if name == "Engine":
        from . import engine
        return engine.Engine
    if name in ("Translator", "RunConfig"):
        from . import translator
        return getattr(translator, name)
    if name in ("greedy_translate", "beam_translate", "SearchConfig", "max_out_length"):
        from . import search
        return getattr(search, name)
    raise AttributeError(name)
