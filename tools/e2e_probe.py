import ctypes as C, time, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_1603_07846_b200 import _lib as L, net as PN
from workloads import configs, generate
cfg = sys.argv[1] if len(sys.argv) > 1 else "cifar10"
torch.cuda.set_device(0)
net_cfg = configs.get(cfg); b = bench.PER_GPU_BATCH[cfg]
n = PN.Net(PN.Cluster(0, 1, 0, None), net_cfg, b)
n.set_updater(configs.UPDATERS[cfg]); n.set_params(bench.init_params(PN, n, net_cfg)); n.enable_graph(True)
xs = [torch.from_numpy(np.ascontiguousarray(generate.batch(net_cfg, b, t)[0])).pin_memory() for t in range(8)]
ls = [torch.from_numpy(np.ascontiguousarray(generate.batch(net_cfg, b, t)[1])).pin_memory() for t in range(8)]
loss_h = torch.zeros(200).pin_memory()
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for mode in ("sync", "async", "async", "sync"):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); tq = 0
    for t in range(100):
        j = t % 8
        a = time.perf_counter()
        if mode == "async":
            L.sg_train_one_batch_host_async(n.h, n.upd, t, C.c_void_p(xs[j].data_ptr()), C.c_void_p(ls[j].data_ptr()), C.c_void_p(loss_h[t:].data_ptr()), sp)
        else:
            lh = C.c_float()
            L.sg_train_one_batch_host(n.h, n.upd, t, C.c_void_p(xs[j].data_ptr()), C.c_void_p(ls[j].data_ptr()), C.byref(lh), sp)
        tq += time.perf_counter() - a
    t1 = time.perf_counter()
    n.sync(); torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(mode, f"per-call host {tq/100*1e6:.1f} us, loop {(t1-t0)/100*1e6:.1f} us, total {(t2-t0)/100*1e6:.1f} us/step")
