"""mvgs — B200-native batched multi-view differentiable rasterizer with fused
multi-view ADC statistics (arXiv 2506.12727).  The compute path is
libmvgs.so (csrc/, sm_100a CUDA) behind the C ABI of include/mvgs.h;
`mvgs.py` is the thin ctypes binding."""
from .mvgs import (Rasterizer, adc_stats, create, destroy, export_lists, export_pairs, preprocess, query,
                   render_bwd, render_fwd, reserve, MvgsError)

__all__ = ["Rasterizer", "adc_stats", "create", "destroy", "export_lists", "export_pairs", "preprocess", "query",
           "render_bwd", "render_fwd", "reserve", "MvgsError"]
