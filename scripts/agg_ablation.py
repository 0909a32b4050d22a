"""The paper's server-traffic question on B200 (PAPER.md P:73, P:203, P:221-222,
§4.3): cost of the cross-rank aggregation step of a C3-law round for

  * peer          — per-rank fp64 partials, one cooperative kernel reduce-scattering them over
                    peer memory, finalizing and all-gathering θ_new (FL_AGG_PEER);
  * unaggregated  — every client model shipped to the server rank, which averages all of them
                    (FL_AGG_UNAGGREGATED, the ablation without partial aggregation);
  * nccl          — per-rank partial [S‖N] -> ncclAllReduce -> finalize (1-rank communicator here:
                    NCCL refuses two ranks on one GPU, so only its world-1 cost is measured).

Two ranks are contexts of one process on disjoint SM partitions of the one B200 (green contexts),
so "peer memory" is the same HBM: the bytes each mode moves between ranks are exact (xfer_bytes),
the times are HBM-bound stand-ins for NVLink transfers.  Prints one JSON object.
"""
import json
import os
import sys
import threading

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2306_17453_b200 as fl  # noqa: E402
import synth  # noqa: E402

CLIENTS = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
ROUNDS = 4

wl = synth.preset("C3", E=1)
sizes_all = synth.client_sizes(wl)
ids = np.sort(np.random.default_rng(5).choice(10000, size=CLIENTS, replace=False))
_, x, y = synth.population(wl, sizes_all, clients=ids)
sizes = sizes_all[ids]
xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y.astype(np.int32)).cuda()
theta = synth.init_params("cnn")
cohort = np.arange(CLIENTS)


def cfg(**kw):
    return fl.Config(model="cnn", batch_size=32, local_epochs=1, lr=wl.lr, **kw)


def two_ranks(mode):
    rs = [fl.fl_round_init(cfg(rank=r, world_size=2, sm_count=s, agg_mode=mode), sizes, xd, yd, theta)
          for r, s in ((0, 74), (1, -74))]
    blobs = [rs[0].fl_peer_export(CLIENTS), rs[1].fl_peer_export(0)]
    for r in rs:
        r.fl_peer_connect(blobs)
    out = [[], []]

    def w(i):
        for k in range(ROUNDS + 1):
            out[i].append(rs[i].fl_round(cohort, round_index=k))

    th = [threading.Thread(target=w, args=(i,)) for i in range(2)]
    [t.start() for t in th]
    [t.join() for t in th]
    theta_new = [r.fl_get_global_params() for r in rs]
    assert np.array_equal(theta_new[0], theta_new[1])
    for r in rs:
        r.close()
    per = [[s for s in out[i][1:]] for i in range(2)]
    return {"agg_ms_rank": [float(np.median([s["agg_ms"] for s in per[i]])) for i in range(2)],
            "xfer_bytes_rank": [int(per[i][-1]["xfer_bytes"]) for i in range(2)],
            "clients_rank": [int(per[i][-1]["clients_local"]) for i in range(2)],
            "round_ms_max": float(np.median([max(per[0][k]["round_ms"], per[1][k]["round_ms"]) for k in range(ROUNDS)])),
            # a rank's agg_ms includes waiting for the slower rank; the later rank's is the step itself
            "agg_after_last_train_ms": float(min(np.median([s["agg_ms"] for s in per[i]]) for i in range(2)))}


res = {"workload": f"{CLIENTS} C3-law CIFAR clients, E=1, two ranks on 74+74 SMs of one B200; "
                   f"median of {ROUNDS} rounds; P = {fl.fl_n_params('cnn')}"}
for mode in ("peer", "unaggregated"):
    res[mode] = two_ranks(mode)
# world 1: the fused accumulate+finalize, the peer kernel, and NCCL through a 1-rank communicator
for name, kw in (("fused_world1", {}), ("peer_world1", {"agg_mode": "peer"}),
                 ("nccl_world1", {"nccl_unique_id": fl.fl_nccl_unique_id()})):
    c = fl.fl_round_init(cfg(**kw), sizes, xd, yd, theta)
    if name == "peer_world1":
        c.fl_peer_connect([c.fl_peer_export(0)])
    st = [c.fl_round(cohort, round_index=k) for k in range(ROUNDS + 1)][1:]
    res[name] = {"agg_ms": float(np.median([s["agg_ms"] for s in st])), "allreduce_ms":
                 float(np.median([s["allreduce_ms"] for s in st])), "xfer_bytes": int(st[-1]["xfer_bytes"])}
    c.close()
print(json.dumps(res, indent=1))
