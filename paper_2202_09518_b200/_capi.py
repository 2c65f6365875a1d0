"""ctypes binding of the C-ABI in ``include/oocnmf_b200.h`` (liboocnmf_b200.so).

The shared library is the product; this module only declares argument types. There is no
Python or CPU fallback: if the library is missing, importing it raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# (OOCNMF_LIB_PATH: developer A/B of two builds of the same library on one box)
LIB_PATH = os.environ.get("OOCNMF_LIB_PATH") or os.path.join(_HERE, "lib", "liboocnmf_b200.so")

u64 = C.c_uint64
i32 = C.c_int32
dbl = C.c_double
pd = C.POINTER(C.c_double)
pf = C.POINTER(C.c_float)
pu = C.POINTER(C.c_uint64)
vp = C.c_void_p


class Config(C.Structure):
    _fields_ = [("k", u64), ("eta", dbl), ("max_iters", u64), ("error_check_interval", u64),
                ("epsilon", dbl), ("seed", u64), ("init", i32), ("error_mode", i32)]


class Info(C.Structure):
    _fields_ = [("h_update_s", dbl), ("w_update_s", dbl), ("allreduce_s", dbl), ("error_check_s", dbl),
                ("io_s", dbl), ("total_s", dbl), ("flops", dbl), ("peak_resident_bytes", u64),
                ("iterations_run", u64), ("converged", i32), ("reserved", i32), ("n_trace", u64),
                ("aht_pass_ms", dbl), ("wta_pass_ms", dbl), ("aht_pass_launches", u64),
                ("wta_pass_launches", u64), ("gpu_launches", u64), ("h2d_bytes", dbl),
                ("fused_pass_ms", dbl), ("fused_pass_launches", u64), ("h2d_batches", u64)]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_ if name != "reserved"}


class SelectionConfig(C.Structure):
    _fields_ = [("k_min", u64), ("k_max", u64), ("n_perturbations", u64), ("delta", dbl), ("sil_threshold", dbl),
                ("nmf", Config), ("seed", u64)]


class KRecord(C.Structure):
    _fields_ = [("k", u64), ("valid", i32), ("reserved", i32), ("runs_used", u64), ("min_silhouette", dbl),
                ("mean_silhouette", dbl), ("mean_relative_error", dbl), ("iterations", u64)]


pi64 = C.POINTER(C.c_int64)


class MemoryReport(C.Structure):
    _fields_ = [("a_slab_bytes", u64), ("store_peak_bytes", u64), ("factor_bytes", u64),
                ("intermediate_bytes", u64), ("peak_bytes", u64), ("min_n_b", u64), ("feasible", i32),
                ("in_core", i32)]

_SIGS = {
    "oocnmf_last_error": ([], C.c_char_p),
    "oocnmf_abi_version": ([], C.c_int),
    "oocnmf_device_count": ([C.POINTER(C.c_int)], C.c_int),
    "oocnmf_init_factors_host": ([u64, u64, u64, u64, pd, pd], C.c_int),
    "oocnmf_counter_uniform": ([u64, u64, u64, u64, pd], C.c_int),
    "oocnmf_split_even": ([u64, u64, pu], C.c_int),
    "oocnmf_ctx_create": ([C.c_int, C.POINTER(vp)], C.c_int),
    "oocnmf_comm_unique_id": ([C.c_char_p], C.c_int),
    "oocnmf_ctx_create_comm": ([C.c_int, C.c_int, C.c_int, C.c_char_p, C.POINTER(vp)], C.c_int),
    "oocnmf_ctx_destroy": ([vp], C.c_int),
    "oocnmf_ctx_rank": ([vp, C.POINTER(C.c_int), C.POINTER(C.c_int)], C.c_int),
    "oocnmf_ctx_paths": ([vp, C.POINTER(C.c_int)], C.c_int),
    "oocnmf_set_problem": ([vp, u64, u64, u64, u64, u64], C.c_int),
    "oocnmf_load_dense_f64": ([vp, pd, u64], C.c_int),
    "oocnmf_load_dense_f32": ([vp, pf, u64], C.c_int),
    "oocnmf_load_dense_device_f32": ([vp, vp, u64], C.c_int),
    "oocnmf_generate_dense_uniform": ([vp, u64, u64], C.c_int),
    "oocnmf_load_csr_f64": ([vp, pu, pu, pd], C.c_int),
    "oocnmf_generate_csr_uniform": ([vp, dbl, u64], C.c_int),
    "oocnmf_attach_host_dense_f32": ([vp, vp, u64, u64], C.c_int),
    "oocnmf_host_register": ([vp, u64], C.c_int),
    "oocnmf_host_unregister": ([vp], C.c_int),
    "oocnmf_download_dense_f32": ([vp, vp], C.c_int),
    "oocnmf_csr_nnz": ([vp, pu], C.c_int),
    "oocnmf_download_csr": ([vp, pu, pu, pd], C.c_int),
    "oocnmf_set_factors_f64": ([vp, pd, pd], C.c_int),
    "oocnmf_get_factors_f64": ([vp, pd, pd], C.c_int),
    "oocnmf_gather_w_f64": ([vp, pd], C.c_int),
    "oocnmf_solve": ([vp, C.POINTER(Config), pu, pd, u64, C.POINTER(Info)], C.c_int),
    "oocnmf_products_f64": ([vp, pd, pd, pd, pd], C.c_int),
    "oocnmf_sq_norm": ([vp, pd], C.c_int),
    "oocnmf_problem_dims": ([vp, pu, pu, pu, pu, pu], C.c_int),
    "oocnmf_set_problem_cols": ([vp, u64, u64, u64, u64, u64], C.c_int),
    "oocnmf_memory_estimate": ([u64, u64, u64, C.c_int, C.c_int, dbl, u64, C.c_int, C.POINTER(MemoryReport)], C.c_int),
    "oocnmf_gather_h_f64": ([vp, pd], C.c_int),
    "oocnmf_set_rank": ([vp, u64], C.c_int),
    "oocnmf_perturb": ([vp, dbl, u64], C.c_int),
    "oocnmf_set_local": ([vp, C.c_int], C.c_int),
    "oocnmf_allreduce_sum_f64": ([vp, pd, u64], C.c_int),
    "oocnmf_allreduce_f64": ([vp, pd, u64, C.c_int], C.c_int),
    "oocnmf_barrier": ([vp], C.c_int),
    "oocnmf_comm_stats": ([vp, pu, pu, pd], C.c_int),
    "oocnmf_comm_reset_stats": ([vp], C.c_int),
    "oocnmf_set_comm_timeout": ([vp, dbl], C.c_int),
    "oocnmf_ctx_create_group": ([C.c_int, C.POINTER(C.c_int), C.POINTER(vp)], C.c_int),
    "oocnmf_select_k": ([vp, C.POINTER(SelectionConfig), C.POINTER(KRecord), u64, pd, pi64, C.c_char_p, u64],
                        C.c_int),
    "oocnmf_cluster_silhouette": ([pd, u64, u64, u64, pd, pd, pd, pd, pu, pi64], C.c_int),
    "oocnmf_pearson_correlation": ([pd, u64, u64, pd, u64, pd], C.c_int),
    "oocnmf_pdn1_info": ([C.c_char_p, C.POINTER(i32), C.POINTER(i32), pu, pu, pu], C.c_int),
    "oocnmf_pdn1_read_dense": ([C.c_char_p, u64, u64, u64, u64, pd], C.c_int),
    "oocnmf_pdn1_read_dense_f32": ([C.c_char_p, u64, u64, u64, u64, pf], C.c_int),
    "oocnmf_pdn1_csr_rows_nnz": ([C.c_char_p, u64, u64, pu], C.c_int),
    "oocnmf_pdn1_read_csr_rows": ([C.c_char_p, u64, u64, pu, pu, pd], C.c_int),
    "oocnmf_pdn1_write_dense": ([C.c_char_p, pd, u64, u64, i32], C.c_int),
    "oocnmf_pdn1_write_dense_f32": ([C.c_char_p, pf, u64, u64], C.c_int),
    "oocnmf_pdn1_write_csr": ([C.c_char_p, u64, u64, pu, pu, pd, i32], C.c_int),
    "oocnmf_mtx_info": ([C.c_char_p, C.POINTER(i32), pu, pu, pu], C.c_int),
    "oocnmf_mtx_read": ([C.c_char_p, pd, pu, pu, pd], C.c_int),
    "oocnmf_mtx_write_dense": ([C.c_char_p, pd, u64, u64], C.c_int),
    "oocnmf_mtx_write_csr": ([C.c_char_p, u64, u64, pu, pu, pd], C.c_int),
    "oocnmf_nmf_serial_dense_f64": ([C.c_int, pd, u64, u64, C.POINTER(Config), pd, pd, pd, pd, pu, pd, u64,
                                     C.POINTER(Info)], C.c_int),
    "oocnmf_nmf_serial_dense_f32": ([C.c_int, pf, u64, u64, C.POINTER(Config), pd, pd, pd, pd, pu, pd, u64,
                                     C.POINTER(Info)], C.c_int),
    "oocnmf_nmf_serial_csr_f64": ([C.c_int, pu, pu, pd, u64, u64, C.POINTER(Config), pd, pd, pd, pd, pu, pd,
                                   u64, C.POINTER(Info)], C.c_int),
}

EXPORTS = tuple(_SIGS)

_lib = None


def lib():
    """Load liboocnmf_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                              f"g.build()'` (make -C paper_2202_09518_b200/csrc). There is no CPU fallback.")
        handle = C.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(handle, name)
            fn.argtypes = args
            fn.restype = res
        _lib = handle
    return _lib
