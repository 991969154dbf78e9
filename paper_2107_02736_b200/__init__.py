"""B200-native KDE query path of DEANN (arXiv 2107.02736).

Drop-in for the estimator API of the reference package ``deann``
(/root/reference/pkg/src/deann/__init__.py:8-43, hot-path subset):
``Dataset``, ``KernelFamily``/``KernelSpec``, ``naive_kde``, ``rs_kde``,
``deann``, ``deann_batch``, ``Estimate``/``BatchKde``, ``NeighborList``,
``AnnIndex``/``BruteForceIndex`` (GPU brute force), ``brute_force_knn``, the
inverted-file index (``ivf_build``, ``ivf_query``, ``IvfAnnIndex``), the
permuted sampler (``RspState``, ``rsp_kde``) and DEANN1 files (``load``/``save``).
All arithmetic runs in hand-written sm_100a kernels behind the C-ABI in
``include/deann_b200.h``; see DESIGN.md.
"""

from .ann import AnnIndex, BruteForceIndex, GpuBruteForceIndex, NeighborList, brute_force_knn, knn_batch
from .bandwidth import fit_bandwidth, NoBandwidthError
from .data import (
    Dataset,
    DatasetFormatError,
    PermutedDataset,
    Splits,
    as_gpu_dataset,
    file_info,
    load,
    permute,
    save,
    split,
)
from .distance import DistanceMatrix, NormConsistencyError, batch_sqdist, sqdist, window_sqdist
from .estimators import (
    BatchKde,
    Estimate,
    RspState,
    deann,
    deann_arrays,
    dataset_sha256,
    deann_batch,
    ground_truth,
    kernel_from_distance,
    kernel_pair,
    naive_kde,
    naive_kde_into,
    rs_kde,
    rsp_kde,
)
from .ivf import (
    IvfAnnIndex,
    IvfIndex,
    ivf_build,
    ivf_query,
    ivf_query_batch,
    load_ivf_index,
    recall,
    save_ivf_index,
)
from .kernels import KernelFamily, KernelSpec
from .sampler import PhiloxSampler

__version__ = "0.1.0"

__all__ = [
    "AnnIndex", "BruteForceIndex", "GpuBruteForceIndex", "NeighborList", "brute_force_knn", "knn_batch",
    "fit_bandwidth", "NoBandwidthError", "Dataset", "DatasetFormatError", "PermutedDataset", "permute",
    "as_gpu_dataset", "file_info", "load", "save", "BatchKde",
    "Estimate", "RspState", "rsp_kde", "deann",
    "deann_arrays", "deann_batch", "kernel_from_distance", "naive_kde", "naive_kde_into", "rs_kde",
    "KernelFamily", "KernelSpec", "PhiloxSampler", "IvfIndex", "IvfAnnIndex", "ivf_build", "ivf_query",
    "ivf_query_batch", "recall", "save_ivf_index", "load_ivf_index",
    "DistanceMatrix", "NormConsistencyError", "batch_sqdist", "sqdist", "window_sqdist",
    "Splits", "split", "kernel_pair", "ground_truth", "dataset_sha256",
]
