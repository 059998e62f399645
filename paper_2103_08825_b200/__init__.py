"""sb200 -- B200-native (sm_100a) multistep stencil sweep.

Drop-in for the hot path of the reference package ``stencilbench``
(arXiv 2103.08825): stencil shape and coefficients, input grid and timestep
count in, output grid out.  Python host code drives hand-written CUDA kernels
through the C ABI in ``include/sb200.h`` (ctypes); there is no CPU fallback.

Public surface:
  core     -- StencilSpec mirror, presets, BASELINE configs (C1-C5)
  plan     -- Plan (device-resident problem), sweep() grid-in/grid-out
  kernels  -- METHODS-compatible b200_step, jam_sweep-compatible b200_sweep,
              register() for the reference's METHODS registry
  grid     -- GridBuffer mirror (NATURAL / BLOCK_TRANSPOSE / DLT storage)
  transpose-- to/from_block_transpose, to/from_dlt on the GPU
  harness  -- the reference's run_benchmark contract for the b200 methods
  slab     -- multi-GPU slab decomposition with halo exchange (overlapped in 2D/3D)
"""

from .core import (CONFIGS, GridError, SpecError, StencilSpec, config_spec,  # noqa: F401
                   flops_per_point, make_stencil_spec)

__version__ = "0.1.0"


def sweep(*args, **kwargs):
    from .plan import sweep as _sweep
    return _sweep(*args, **kwargs)
