"""B200-native (sm_100a) Sub-R-HOSVD / Sub-R-RtL-HT engine.

The compute path is ``libsrtt_b200.so`` (hand-written CUDA kernels behind the
C-ABI in ``include/srtt_b200.h``); :mod:`.srtt` mirrors the reference's API
on top of it.
"""
from .srtt import (  # noqa: F401
    DimensionTree, ExecPolicy, Handle, HTuckerDecomposition, HtSubsampleReport, InvalidArgument, JobError,
    OutOfRange, SubsampleReport, TuckerDecomposition, default_handle, extract_fibers, extract_group_fibers,
    multi_ttm_core, node_sample_counts, range_basis_of_sketch, root_transfer, sample_indices, sketch,
    sliced_core, pick_slice_mode, stream_normals, sub_r_hosvd, sub_r_rtl_ht, transfer_tensor, uniform_node_ranks,
    reconstruct, ht_reconstruct, rel_error, tucker_rel_error, ht_rel_error,
    IoError, read_tensor, write_tensor, tensor_file_info, read_htucker, write_htucker,
)
