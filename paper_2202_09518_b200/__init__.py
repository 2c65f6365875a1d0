"""B200-native Frobenius multiplicative-update NMF (the hot path of pyDNMF-GPU, arXiv 2202.09518).

The product is ``lib/liboocnmf_b200.so`` (C-ABI: ``include/oocnmf_b200.h``; C++ host core:
``include/oocnmf/*.hpp``). This package is its Python front-end, mirroring the reference's
``oocnmf::`` API names.
"""
from .nmf import (  # noqa: F401
    CollectiveStats,
    ColumnClusters,
    CommError,
    Context,
    CsrMatrix,
    DataError,
    DeviceError,
    DistComm,
    FactorInit,
    IoError,
    KRecord,
    NmfConfig,
    NmfResult,
    PartitionPlan,
    PhaseCounters,
    PhaseTag,
    SelectionConfig,
    SelectionReport,
    ShapeError,
    StoreConfig,
    StoreCounters,
    StoreError,
    Strategy,
    check,
    choose_strategy,
    cluster_columns,
    counter_uniform,
    device_count,
    init_factors,
    make_plan,
    memory_estimate,
    nmf_distributed,
    nmf_serial,
    pearson_correlation_matrix,
    run_distributed_threads,
    perturb_dense,
    perturb_sparse,
    select_k,
    spawn_group,
    select_k_distributed,
    split_even,
)

from .io import Pdn1File, read_matrix, read_mtx, read_pdn1, write_mtx, write_pdn1  # noqa: F401,E402

__version__ = "0.1.0"
