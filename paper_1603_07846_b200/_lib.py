"""Thin ctypes binding of include/singa_b200.h (argument marshalling only).

Every ``sg_*`` function of the C ABI is exposed under the same name; a nonzero
status raises :class:`SingaError` carrying ``sg_last_error()``.  There is no
fallback: if the shared library is missing the import fails loudly.
"""

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SG_LIB") or os.path.join(_HERE, "libsinga_b200.so")  # SG_LIB: A/B of two builds

SG_OK = 0
ERRORS = {
    -1: "SG_ERR_INVALID_ARG", -2: "SG_ERR_DIMENSION", -3: "SG_ERR_PARTITION", -4: "SG_ERR_CONFIG",
    -5: "SG_ERR_SEQUENCE", -6: "SG_ERR_PROTOCOL", -7: "SG_ERR_DIVERGED", -8: "SG_ERR_LABEL",
    -9: "SG_ERR_CUDA", -10: "SG_ERR_NCCL", -11: "SG_ERR_OOM", -12: "SG_ERR_UNSUPPORTED",
}
KINDS = {"conv": 1, "pool_max": 2, "pool_avg": 3, "relu": 4, "sigmoid": 5, "lrn": 6, "ip": 7,
         "softmax_ce": 8, "euclidean": 9, "input": 20, "concat": 21, "slice": 22}
KIND_NAMES = {v: k for k, v in KINDS.items()}


class SingaError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.name = ERRORS.get(code, str(code))


class ConvDesc(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("N", "H", "W", "C", "Co", "R", "S", "stride", "pad")]


class PoolDesc(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("N", "H", "W", "C", "kernel", "stride", "pad", "mode")]


class LrnDesc(C.Structure):
    _fields_ = [("pixels", C.c_int64), ("C", C.c_int32), ("size", C.c_int32),
                ("alpha", C.c_float), ("beta", C.c_float), ("k", C.c_float)]


class ClusterCfg(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world_size", C.c_int32), ("device", C.c_int32),
                ("nworker_groups", C.c_int32), ("workers_per_group", C.c_int32),
                ("nserver_groups", C.c_int32), ("servers_per_group", C.c_int32),
                ("nccl_id", C.c_uint8 * 128), ("exercise_collectives", C.c_int32)]


class LayerCfg(C.Structure):
    _fields_ = [("name", C.c_char_p), ("kind", C.c_int32), ("partition_dim", C.c_int32),
                ("num_output", C.c_int32), ("kernel", C.c_int32), ("stride", C.c_int32), ("pad", C.c_int32),
                ("lrn_size", C.c_int32), ("lrn_alpha", C.c_float), ("lrn_beta", C.c_float), ("lrn_k", C.c_float),
                ("lr_scale", C.c_float), ("wd_scale", C.c_float)]


class NetCfg(C.Structure):
    _fields_ = [("nlayers", C.c_int32), ("layers", C.POINTER(LayerCfg)), ("batch", C.c_int32),
                ("in_c", C.c_int32), ("in_h", C.c_int32), ("in_w", C.c_int32), ("num_classes", C.c_int32)]


class LayerInfo(C.Structure):
    _fields_ = [("name", C.c_char * 64), ("kind", C.c_int32), ("partition_dim", C.c_int32),
                ("is_connection", C.c_int32), ("src", C.c_int32),
                ("global_shape", C.c_int64 * 4), ("local_shape", C.c_int64 * 4), ("local_offset", C.c_int64 * 4),
                ("ld", C.c_int64), ("nblocks", C.c_int32), ("tf32_data", C.c_int32), ("tf32_grad", C.c_int32)]


class ParamInfo(C.Structure):
    _fields_ = [("name", C.c_char * 64), ("layer", C.c_int32), ("split_dim", C.c_int32),
                ("rows", C.c_int64), ("cols", C.c_int64), ("local_col_off", C.c_int64), ("local_cols", C.c_int64),
                ("bucket", C.c_int32), ("bucket_off", C.c_int64), ("internal_size", C.c_int64)]


class ShardRange(C.Structure):
    _fields_ = [("param", C.c_int32), ("bucket", C.c_int32), ("owner_rank", C.c_int32),
                ("param_off", C.c_int64), ("bucket_off", C.c_int64), ("len", C.c_int64)]


class UpdaterCfg(C.Structure):
    _fields_ = [("base_lr", C.c_float), ("momentum", C.c_float), ("weight_decay", C.c_float),
                ("grad_scale", C.c_float), ("lr_policy", C.c_int32), ("gamma", C.c_float), ("step_size", C.c_int32),
                ("type", C.c_int32), ("eps", C.c_float)]


P = C.c_void_p
I32, I64, F32 = C.c_int32, C.c_int64, C.c_float
PI32, PI64 = C.POINTER(C.c_int32), C.POINTER(C.c_int64)

# name -> argtypes (restype is always int32 status unless listed in _RESTYPES)
SIGS = {
    "sg_partition_range": [I64, I32, I32, PI64, PI64],
    "sg_op_gemm": [P, I32, P, I32, P, I32, I32, I32, P],
    "sg_conv_out_shape": [C.POINTER(ConvDesc), PI32, PI32],
    "sg_op_conv_forward": [C.POINTER(ConvDesc), P, P, P, P, P],
    "sg_op_conv_backward": [C.POINTER(ConvDesc), P, P, P, P, P, P, P],
    "sg_op_ip_forward": [P, P, P, P, I32, I32, I32, P],
    "sg_op_ip_backward": [P, P, P, P, P, P, I32, I32, I32, P],
    "sg_pool_out_shape": [C.POINTER(PoolDesc), PI32, PI32],
    "sg_op_pool_forward": [C.POINTER(PoolDesc), P, P, P, P],
    "sg_op_pool_backward": [C.POINTER(PoolDesc), P, P, P, P],
    "sg_op_pool_argmax": [C.POINTER(PoolDesc), P, P, P],
    "sg_op_lrn_forward": [C.POINTER(LrnDesc), P, P, P, P],
    "sg_op_lrn_backward": [C.POINTER(LrnDesc), P, P, P, P, P, P],
    "sg_op_neuron_forward": [I32, P, P, I64, P],
    "sg_op_neuron_backward": [I32, P, P, P, I64, P],
    "sg_op_softmax_ce": [P, P, I32, I32, I32, P, P, P, P],
    "sg_op_euclidean": [P, P, I32, I32, I32, P, P, P],
    "sg_op_sgd_momentum": [P, P, P, I64, F32, F32, F32, F32, P],
    "sg_op_adagrad": [P, P, P, I64, F32, F32, F32, F32, P],
    "sg_get_unique_id": [C.POINTER(C.c_uint8 * 128)],
    "sg_cluster_create": [C.POINTER(ClusterCfg), C.POINTER(P)],
    "sg_cluster_framework": [P, C.POINTER(C.c_char_p)],
    "sg_cluster_destroy": [P],
    "sg_plan_create": [C.POINTER(NetCfg), I32, I32, C.POINTER(P)],
    "sg_layer_cost": [I64, I64, I64, I64, I32, I32, PI64],
    "sg_recommend_plan": [C.POINTER(NetCfg), I32, PI32, PI32, PI64, PI64],
    "sg_plan_destroy": [P],
    "sg_plan_num_layers": [P, PI32],
    "sg_plan_layer_info": [P, I32, C.POINTER(LayerInfo)],
    "sg_plan_num_params": [P, PI32],
    "sg_plan_param_info": [P, I32, C.POINTER(ParamInfo)],
    "sg_plan_num_buckets": [P, PI32, PI64],
    "sg_plan_shard_map": [P, C.POINTER(ShardRange), I32, PI32],
    "sg_net_create": [P, C.POINTER(NetCfg), C.POINTER(P)],
    "sg_net_destroy": [P],
    "sg_net_plan": [P, C.POINTER(P)],
    "sg_param_set_value": [P, I32, P],
    "sg_param_get_value": [P, I32, P],
    "sg_param_get_grad": [P, I32, P],
    "sg_param_get_history": [P, I32, P],
    "sg_param_get_working": [P, I32, P],
    "sg_updater_create": [P, C.POINTER(UpdaterCfg), C.POINTER(P)],
    "sg_updater_destroy": [P],
    "sg_train_one_batch": [P, P, I64, P, P, P, P],
    "sg_train_one_batch_host": [P, P, I64, P, P, P, P],
    "sg_train_one_batch_host_async": [P, P, I64, P, P, P, P],
    "sg_net_set_input": [P, P, P, P],
    "sg_net_collect": [P, I32, P],
    "sg_layer_compute_feature": [P, I32, P],
    "sg_layer_compute_gradient": [P, I32, P],
    "sg_net_update": [P, P, I32, I64, P],
    "sg_net_loss": [P, P, P],
    "sg_net_sync": [P],
    "sg_net_enable_graph": [P, I32],
    "sg_net_set_fusion": [P, I32],
    "sg_net_set_exchange": [P, I32],
    "sg_net_set_overlap": [P, I32],
    "sg_net_last_launch_count": [P, PI64],
    "sg_net_profile": [P, I32],
    "sg_net_op_times": [P, C.POINTER(C.c_double), PI64, I32, PI32, I32],
    "sg_net_op_timeline": [P, C.POINTER(C.c_double), C.POINTER(C.c_double), I32, PI32],
    "sg_blob_size": [P, I32, I32, C.POINTER(C.c_size_t)],
    "sg_blob_get": [P, I32, I32, P, C.c_size_t, P],
    "sg_blob_set": [P, I32, I32, P, C.c_size_t, P],
    "sg_server_sync": [P, C.POINTER(UpdaterCfg), I64, P, P, P, I64, P],
    "sg_peer_sync_create": [P, I64, C.POINTER(P), C.POINTER(P), C.POINTER(P), C.POINTER(P)],
    "sg_nvls_sync_create": [P, I64, C.POINTER(P), C.POINTER(P), C.POINTER(P), C.POINTER(P)],
    "sg_peer_sync_step": [P, C.POINTER(UpdaterCfg), I64, P],
    "sg_nvls_sync_step": [P, C.POINTER(UpdaterCfg), I64, P],
    "sg_peer_sync_destroy": [P],
    "sg_nvls_sync_destroy": [P],
}
_RESTYPES = {"sg_last_error": C.c_char_p, "sg_abi_version": C.c_int32}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1603_07846_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, rt in _RESTYPES.items():
        getattr(lib, name).restype = rt
        getattr(lib, name).argtypes = []
    for name, args in SIGS.items():
        f = getattr(lib, name)
        f.restype = C.c_int32
        f.argtypes = args
    return lib


lib = _load()


def last_error():
    return lib.sg_last_error().decode()


def _wrap(name):
    f = getattr(lib, name)

    def call(*args):
        st = f(*args)
        if st != SG_OK:
            raise SingaError(st, last_error())
        return st
    call.__name__ = name
    return call


for _n in SIGS:
    globals()[_n] = _wrap(_n)


def sg_abi_version():
    return lib.sg_abi_version()


def sg_last_error():
    return last_error()
