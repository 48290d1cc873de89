"""B200-native streaming-TTS serving hot path (VoxServe, arxiv 2602.00269).

Drop-in executor behind the reference's model-execution interface
(speechserve.model_api) driven by its unchanged streaming-aware scheduler.
Device code: csrc/*.cu (sm_100a) behind the C-ABI in include/voxb200.h.
"""

__version__ = "0.1.0"
