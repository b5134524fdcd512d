"""B200-native m-Cubes VEGAS iteration (arXiv 2202.01753).

A drop-in for the sampling path of the reference's header-only ``mcubes``
library: the same API (``integrate``, ``v_sample``, ``v_sample_no_adjust``,
``RunConfig``, ``Grid``, ...) backed by hand-written sm_100a kernels in
``libmcubes_b200.so``.  See DESIGN.md and INTEGRATION.md.
"""
from .mcubes import (  # noqa: F401
    BinAccumulator,
    BinUpdate,
    Checkpoint,
    Combined,
    Context,
    CudaError,
    EstimateVariance,
    Grid,
    IntegrandSpec,
    IntegrationResult,
    IterationResult,
    IterationView,
    NonFiniteSample,
    Run,
    RunConfig,
    SampleOutcome,
    SetupParams,
    Variant,
    check_convergence,
    default_context,
    integrate,
    make_fA,
    make_fB,
    make_integrand,
    make_suite_integrand,
    make_table_integrand,
    parse_variant,
    reference_value,
    set_batch_size,
    set_device,
    setup,
    test_integrand,
    v_sample,
    v_sample_no_adjust,
    variant_name,
    weighted_estimate,
)

__all__ = [n for n in dir() if not n.startswith("_")]
