"""B200-native (sm_100a) M-step solver of arXiv 1905.13408 (cryomap::m_step drop-in).

The product is libcm.so (include/cm_api.h), built from csrc/ by
``python -m paper_1905_13408_b200.build``. This package is the Python mirror
of the reference interface (regularizer.hpp / params.hpp / fourier.hpp) over
that C ABI; synth.py generates the synthetic benchmark inputs.
"""
from .regularizer import (  # noqa: F401
    AccumulatorPair, Context, DataScales, DeviceError, Error, GridMismatch, InvalidArgument,
    MStepTraceRow, Multipliers, NonHermitianAccumulator, NonHermitianInput, NonPositiveScale,
    ObjectiveValue, RegConfig, Refresh, SolveStats, StepDiverged, StepRule, WeightFields,
    compute_weights, context, data_gradient, derive_config, em_m_step, fft3, fft3_centered, m_step,
    penalized_objective,
    prox_l1, scale_data, smoothed_tv_gradient, smoothed_tv_value, validate_reg_config,
)

from . import slab  # noqa: F401,E402
from .backproject import (  # noqa: F401,E402
    BackprojectInput, backproject_accumulate, backproject_into, e_step, posterior_entries,
    sparse_entries,
    set_particles,
)
from .slab import SlabContext, SlabPlan  # noqa: F401,E402

__version__ = "0.1.0"
