"""Workload definitions (pure data, no arithmetic of the method).

These are the NeuralNet configurations of BASELINE.json ``configs`` as read in
SURVEY.md §8.0.  Both the oracle (``oracle/``) and the CUDA path consume the same
dictionaries; neither derives anything from the other.  Every layer is a chain
element whose single source layer is the previous entry (§4.1.1:
"each layer records its own source layers"; all configs here are single-path
feed-forward nets).

Layer dict keys:
  name, kind in {conv, pool_max, pool_avg, relu, sigmoid, lrn, ip, softmax_ce,
  euclidean}, plus kind-specific hyper-parameters, and ``partition_dim``
  (0 = batch dim / data parallel, 1 = feature dim / model parallel;
  P:479-484 §5.3).  Layers without ``partition_dim`` inherit their source's
  ("consistent with source layers").
"""

import copy

# cuda-convnet CIFAR-10 "18%" shape with an LRN in each of the 3 blocks
# (BASELINE configs[1] "conv-pool-LRN x3").
CIFAR10 = {
    "name": "cifar10",
    "input": {"c": 3, "h": 32, "w": 32},
    "num_classes": 10,
    "layers": [
        {"name": "conv1", "kind": "conv", "num_output": 32, "kernel": 5, "stride": 1, "pad": 2, "partition_dim": 0},
        {"name": "pool1", "kind": "pool_max", "kernel": 3, "stride": 2, "pad": 0},
        {"name": "relu1", "kind": "relu"},
        {"name": "norm1", "kind": "lrn", "size": 3, "alpha": 5e-5, "beta": 0.75, "k": 1.0},
        {"name": "conv2", "kind": "conv", "num_output": 32, "kernel": 5, "stride": 1, "pad": 2},
        {"name": "relu2", "kind": "relu"},
        {"name": "pool2", "kind": "pool_avg", "kernel": 3, "stride": 2, "pad": 0},
        {"name": "norm2", "kind": "lrn", "size": 3, "alpha": 5e-5, "beta": 0.75, "k": 1.0},
        {"name": "conv3", "kind": "conv", "num_output": 64, "kernel": 5, "stride": 1, "pad": 2},
        {"name": "relu3", "kind": "relu"},
        {"name": "pool3", "kind": "pool_avg", "kernel": 3, "stride": 2, "pad": 0},
        {"name": "norm3", "kind": "lrn", "size": 3, "alpha": 5e-5, "beta": 0.75, "k": 1.0},
        {"name": "ip1", "kind": "ip", "num_output": 10},
        {"name": "loss", "kind": "softmax_ce"},
    ],
}

# MLP 784-256-10 with the paper's running-example logistic hidden layer
# (BASELINE configs[0]; "applies non-linear (logistic) transformations").
MLP = {
    "name": "mlp",
    "input": {"d": 784},
    "num_classes": 10,
    "layers": [
        {"name": "ip1", "kind": "ip", "num_output": 256, "partition_dim": 0},
        {"name": "sig1", "kind": "sigmoid"},
        {"name": "ip2", "kind": "ip", "num_output": 10},
        {"name": "loss", "kind": "softmax_ce"},
    ],
}


def alexnet(hybrid=True, pool5=True):
    """convnet-benchmarks AlexNet.

    ``hybrid``: conv side partition_dim 0, fc6..fc8 partition_dim 1, loss dim 0
    ("data parallelism for layers before the first fully connected layer,
    and then model parallelism").  ``pool5=False`` is the variant that makes
    fc6 have 13*13*256*4096 = 177,209,344 weights (reading A17).
    """
    fc_dim = 1 if hybrid else 0
    layers = [
        {"name": "conv1", "kind": "conv", "num_output": 64, "kernel": 11, "stride": 4, "pad": 2, "partition_dim": 0},
        {"name": "relu1", "kind": "relu"},
        {"name": "pool1", "kind": "pool_max", "kernel": 3, "stride": 2, "pad": 0},
        {"name": "conv2", "kind": "conv", "num_output": 192, "kernel": 5, "stride": 1, "pad": 2},
        {"name": "relu2", "kind": "relu"},
        {"name": "pool2", "kind": "pool_max", "kernel": 3, "stride": 2, "pad": 0},
        {"name": "conv3", "kind": "conv", "num_output": 384, "kernel": 3, "stride": 1, "pad": 1},
        {"name": "relu3", "kind": "relu"},
        {"name": "conv4", "kind": "conv", "num_output": 256, "kernel": 3, "stride": 1, "pad": 1},
        {"name": "relu4", "kind": "relu"},
        {"name": "conv5", "kind": "conv", "num_output": 256, "kernel": 3, "stride": 1, "pad": 1},
        {"name": "relu5", "kind": "relu"},
    ]
    if pool5:
        layers.append({"name": "pool5", "kind": "pool_max", "kernel": 3, "stride": 2, "pad": 0})
    layers += [
        {"name": "fc6", "kind": "ip", "num_output": 4096, "partition_dim": fc_dim},
        {"name": "relu6", "kind": "relu"},
        {"name": "fc7", "kind": "ip", "num_output": 4096},
        {"name": "relu7", "kind": "relu"},
        {"name": "fc8", "kind": "ip", "num_output": 1000},
        {"name": "loss", "kind": "softmax_ce", "partition_dim": 0},
    ]
    return {"name": "alexnet" + ("" if pool5 else "_nopool5"),
            "input": {"c": 3, "h": 224, "w": 224}, "num_classes": 1000, "layers": layers}


ALEXNET = alexnet()


def autoencoder(widths, name):
    """Deep auto-encoder (P:612-613, 784-1000-500-250-2 stack unrolled into an
    encoder/decoder), sigmoid everywhere except the linear code layer, Euclidean
    loss against the input; every layer partition_dim 1."""
    layers = []
    code = len(widths) // 2
    for i, w in enumerate(widths[1:], start=1):
        layers.append({"name": f"ip{i}", "kind": "ip", "num_output": w, "partition_dim": 1})
        if i != code:
            layers.append({"name": f"sig{i}", "kind": "sigmoid"})
    layers.append({"name": "loss", "kind": "euclidean"})
    return {"name": name, "input": {"d": widths[0]}, "num_classes": 0, "layers": layers}


AE = autoencoder([784, 1000, 500, 250, 2, 250, 500, 1000, 784], "ae")
AE_WIDE = autoencoder([784, 8000, 4000, 2000, 16, 2000, 4000, 8000, 784], "ae_wide")

# Tiny nets used by parity tests at sizes the oracle finishes in seconds.
TINY_CONV = {
    "name": "tiny_conv",
    "input": {"c": 3, "h": 12, "w": 12},
    "num_classes": 5,
    "layers": [
        {"name": "conv1", "kind": "conv", "num_output": 8, "kernel": 3, "stride": 1, "pad": 1, "partition_dim": 0},
        {"name": "pool1", "kind": "pool_max", "kernel": 3, "stride": 2, "pad": 0},
        {"name": "relu1", "kind": "relu"},
        {"name": "norm1", "kind": "lrn", "size": 3, "alpha": 1e-2, "beta": 0.75, "k": 1.0},
        {"name": "conv2", "kind": "conv", "num_output": 8, "kernel": 3, "stride": 1, "pad": 1},
        {"name": "relu2", "kind": "relu"},
        {"name": "pool2", "kind": "pool_avg", "kernel": 3, "stride": 2, "pad": 0},
        {"name": "ip1", "kind": "ip", "num_output": 5},
        {"name": "loss", "kind": "softmax_ce"},
    ],
}

# the paper's ablation baseline: every layer data parallel
ALEXNET_DP = dict(alexnet(hybrid=False), name="alexnet_dp")

NETS = {"mlp": MLP, "cifar10": CIFAR10, "alexnet": ALEXNET, "alexnet_dp": ALEXNET_DP, "ae": AE, "ae_wide": AE_WIDE,
        "tiny_conv": TINY_CONV}

# Updater hyper-parameters per config.
UPDATERS = {
    "mlp": {"base_lr": 0.01, "momentum": 0.9, "weight_decay": 5e-4, "lr_policy": "fixed"},
    "cifar10": {"base_lr": 0.001, "momentum": 0.9, "weight_decay": 0.004, "lr_policy": "fixed"},
    "alexnet": {"base_lr": 0.01, "momentum": 0.9, "weight_decay": 5e-4, "lr_policy": "fixed"},
    "alexnet_dp": {"base_lr": 0.01, "momentum": 0.9, "weight_decay": 5e-4, "lr_policy": "fixed"},
    "ae": {"base_lr": 0.01, "momentum": 0.9, "weight_decay": 0.0, "lr_policy": "fixed"},
    "ae_wide": {"base_lr": 0.01, "momentum": 0.9, "weight_decay": 0.0, "lr_policy": "fixed"},
    "tiny_conv": {"base_lr": 0.01, "momentum": 0.9, "weight_decay": 5e-4, "lr_policy": "fixed"},
}

BATCH = {"mlp": 64, "cifar10": 128, "alexnet": 256, "ae": 256, "ae_wide": 256, "tiny_conv": 8}

JOB_SEED = 160307846


def get(name):
    return copy.deepcopy(NETS[name])


def with_partition(net, dims):
    """Return a copy of ``net`` with partition_dim overridden per layer name."""
    net = copy.deepcopy(net)
    for l in net["layers"]:
        if l["name"] in dims:
            l["partition_dim"] = dims[l["name"]]
    return net
