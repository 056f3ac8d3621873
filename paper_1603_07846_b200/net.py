"""Argument marshalling between the workload dictionaries (workloads/configs.py)
and the C ABI structs.  No computation happens here: every step of the path runs
in libsinga_b200.so (see include/singa_b200.h).
"""

import ctypes as C

import numpy as np

from . import _lib as L


def net_cfg(net, batch):
    """Build an sg_net_cfg (plus the objects it points into, kept alive on it)."""
    layers = net["layers"]
    arr = (L.LayerCfg * len(layers))()
    names = []
    for i, l in enumerate(layers):
        nm = l["name"].encode()
        names.append(nm)
        a = arr[i]
        a.name = nm
        a.kind = L.KINDS[l["kind"]]
        a.partition_dim = l.get("partition_dim", -1)
        a.num_output = l.get("num_output", 0)
        a.kernel = l.get("kernel", 0)
        a.stride = l.get("stride", 1)
        a.pad = l.get("pad", 0)
        a.lrn_size = l.get("size", 0)
        a.lrn_alpha = l.get("alpha", 0.0)
        a.lrn_beta = l.get("beta", 0.0)
        a.lrn_k = l.get("k", 0.0)
        a.lr_scale = l.get("lr_scale", 1.0)
        a.wd_scale = l.get("wd_scale", 1.0)
    inp = net["input"]
    cfg = L.NetCfg()
    cfg.nlayers = len(layers)
    cfg.layers = C.cast(arr, C.POINTER(L.LayerCfg))
    cfg.batch = batch
    if "d" in inp:
        cfg.in_c, cfg.in_h, cfg.in_w = inp["d"], 0, 0
    else:
        cfg.in_c, cfg.in_h, cfg.in_w = inp["c"], inp["h"], inp["w"]
    cfg.num_classes = net["num_classes"]
    cfg._keep = (arr, names)
    return cfg


def updater_cfg(upd, grad_scale=0.0):
    u = L.UpdaterCfg()
    u.base_lr = upd["base_lr"]
    u.momentum = upd["momentum"]
    u.weight_decay = upd["weight_decay"]
    u.grad_scale = grad_scale
    u.lr_policy = 1 if upd.get("lr_policy", "fixed") == "step" else 0
    u.gamma = upd.get("gamma", 1.0)
    u.step_size = upd.get("step_size", 1)
    u.type = 1 if upd.get("type", "sgd_momentum") == "adagrad" else 0
    u.eps = upd.get("eps", 0.0)
    return u


class Plan:
    """Host-only plan (no device needed)."""

    def __init__(self, net, batch, rank=0, world=1, handle=None):
        self._owned = handle is None
        if handle is None:
            self.cfg = net_cfg(net, batch)
            h = C.c_void_p()
            L.sg_plan_create(C.byref(self.cfg), rank, world, C.byref(h))
            handle = h
        self.h = handle

    def close(self):
        if self._owned and self.h:
            L.sg_plan_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def layers(self):
        n = C.c_int32()
        L.sg_plan_num_layers(self.h, C.byref(n))
        out = []
        for i in range(n.value):
            li = L.LayerInfo()
            L.sg_plan_layer_info(self.h, i, C.byref(li))
            out.append({"name": li.name.decode(), "kind": L.KIND_NAMES[li.kind], "partition_dim": li.partition_dim,
                        "is_connection": li.is_connection, "src": li.src,
                        "global_shape": tuple(li.global_shape), "local_shape": tuple(li.local_shape),
                        "local_offset": tuple(li.local_offset), "ld": li.ld, "nblocks": li.nblocks,
                        "tf32_data": bool(li.tf32_data), "tf32_grad": bool(li.tf32_grad)})
        return out

    def params(self):
        n = C.c_int32()
        L.sg_plan_num_params(self.h, C.byref(n))
        out = []
        for i in range(n.value):
            p = L.ParamInfo()
            L.sg_plan_param_info(self.h, i, C.byref(p))
            out.append({"name": p.name.decode(), "layer": p.layer, "split_dim": p.split_dim, "rows": p.rows,
                        "cols": p.cols, "local_col_off": p.local_col_off, "local_cols": p.local_cols,
                        "bucket": p.bucket, "bucket_off": p.bucket_off, "internal_size": p.internal_size})
        return out

    def buckets(self):
        n = C.c_int32()
        L.sg_plan_num_buckets(self.h, C.byref(n), None)
        sizes = (C.c_int64 * max(n.value, 1))()
        L.sg_plan_num_buckets(self.h, C.byref(n), sizes)
        return [sizes[i] for i in range(n.value)]

    def shard_map(self):
        n = C.c_int32()
        L.sg_plan_shard_map(self.h, None, 0, C.byref(n))
        arr = (L.ShardRange * max(n.value, 1))()
        L.sg_plan_shard_map(self.h, arr, n.value, C.byref(n))
        return [(r.param, r.bucket, r.owner_rank, r.param_off, r.bucket_off, r.len) for r in arr[:n.value]]


def param_shape(p):
    """User-layout shape of a Param from sg_param_info (conv W [Co][R][S][C] is reported as rows x cols)."""
    return (p["rows"], p["cols"]) if p["rows"] > 1 or not p["name"].endswith("/b") else (p["cols"],)


class Cluster:
    def __init__(self, rank=0, world=1, device=0, nccl_id=None, exercise_collectives=False):
        cfg = L.ClusterCfg()
        cfg.rank, cfg.world_size, cfg.device = rank, world, device
        cfg.exercise_collectives = 1 if exercise_collectives else 0
        if exercise_collectives and nccl_id is None and world == 1:
            nccl_id = Cluster.unique_id()
        cfg.nworker_groups, cfg.workers_per_group = 1, world
        cfg.nserver_groups, cfg.servers_per_group = 1, world
        if nccl_id is not None:
            C.memmove(cfg.nccl_id, bytes(nccl_id), 128)
        h = C.c_void_p()
        L.sg_cluster_create(C.byref(cfg), C.byref(h))
        self.h = h
        self.rank, self.world = rank, world

    @staticmethod
    def unique_id():
        buf = (C.c_uint8 * 128)()
        L.sg_get_unique_id(C.byref(buf))
        return bytes(buf)

    def close(self):
        if self.h:
            L.sg_cluster_destroy(self.h)
            self.h = None


class Net:
    """A NeuralNet on the cluster's device (handle wrapper)."""

    def __init__(self, cluster, net, batch):
        self.cluster = cluster
        self.cfg = net_cfg(net, batch)
        h = C.c_void_p()
        L.sg_net_create(cluster.h, C.byref(self.cfg), C.byref(h))
        self.h = h
        ph = C.c_void_p()
        L.sg_net_plan(self.h, C.byref(ph))
        self.plan = Plan(None, None, handle=ph)
        self.layer_info = self.plan.layers()
        self.param_info = self.plan.params()
        self.upd = None

    def close(self):
        if self.upd:
            L.sg_updater_destroy(self.upd)
            self.upd = None
        if self.h:
            L.sg_net_destroy(self.h)
            self.h = None

    def set_updater(self, upd, grad_scale=0.0):
        if self.upd:
            L.sg_updater_destroy(self.upd)
        self._ucfg = updater_cfg(upd, grad_scale)
        u = C.c_void_p()
        L.sg_updater_create(self.h, C.byref(self._ucfg), C.byref(u))
        self.upd = u

    def param_index(self):
        return {p["name"]: i for i, p in enumerate(self.param_info)}

    def set_params(self, params):
        for i, p in enumerate(self.param_info):
            v = np.ascontiguousarray(params[p["name"]], dtype=np.float32)
            L.sg_param_set_value(self.h, i, v.ctypes.data_as(C.c_void_p))

    def _export(self, fn, shapes):
        out = {}
        for i, p in enumerate(self.param_info):
            shp = shapes[p["name"]]
            buf = np.empty(shp, np.float32)
            fn(self.h, i, buf.ctypes.data_as(C.c_void_p))
            out[p["name"]] = buf
        return out

    def get_params(self, shapes):
        return self._export(L.sg_param_get_value, shapes)

    def get_grads(self, shapes):
        return self._export(L.sg_param_get_grad, shapes)

    def get_history(self, shapes):
        return self._export(L.sg_param_get_history, shapes)

    def get_working(self, shapes):
        """The working copy the GEMMs read (TF32-RN weights, fp32 biases; reading A19)."""
        return self._export(L.sg_param_get_working, shapes)

    def train_one_batch(self, step, x_ptr, labels_ptr, loss_ptr, stream=None):
        L.sg_train_one_batch(self.h, self.upd, step, x_ptr, labels_ptr, loss_ptr, stream)

    def train_one_batch_host(self, step, x, labels, stream=None):
        loss = C.c_float()
        lp = labels.ctypes.data_as(C.c_void_p) if labels is not None else None
        L.sg_train_one_batch_host(self.h, self.upd, step, x.ctypes.data_as(C.c_void_p), lp, C.byref(loss), stream)
        return loss.value

    def sync(self):
        L.sg_net_sync(self.h)

    def set_exchange(self, mode):
        """0: NCCL chain, 1: fused peer-memory kernel (COLLECTIVE)."""
        L.sg_net_set_exchange(self.h, {"nccl": 0, "p2p": 1}.get(mode, mode))

    def set_fusion(self, on=True):
        L.sg_net_set_fusion(self.h, 1 if on else 0)

    def enable_graph(self, on=True):
        L.sg_net_enable_graph(self.h, 1 if on else 0)

    def launches(self):
        v = C.c_int64()
        L.sg_net_last_launch_count(self.h, C.byref(v))
        return v.value

    def blob_size(self, layer, which):
        v = C.c_size_t()
        L.sg_blob_size(self.h, layer, which, C.byref(v))
        return v.value

    def layer_index(self, name):
        for i, l in enumerate(self.layer_info):
            if l["name"] == name:
                return i
        raise KeyError(name)
