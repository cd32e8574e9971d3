"""CPU profile of the e2e path (Cluster.train_batch_async with host batches) on
one GPU: where the host time per step goes.  Diagnostic only.

    python scripts/e2e_profile.py [config] [steps]
"""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    torch.cuda.set_device(0)
    from paper_1711_06505_b200.runtime import Cluster, ClusterConfig
    B = bench.CONFIGS[name]["B"]
    schema, model, pool = bench.build_workload(name, 0, 1, "bf16")
    cl = Cluster(ClusterConfig(workers=1, servers=1, batch_per_worker=B), model, pool, precision="bf16")
    cl.use_graphs = True
    batches = bench.make_batches(name, schema, 8, seed=1000)
    for b in batches[:4]:
        cl.train_batch_async(b, B)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    t = time.perf_counter()
    pr.enable()
    for i in range(steps):
        cl.train_batch_async(batches[i % len(batches)], B)
    pr.disable()
    cpu = time.perf_counter() - t
    torch.cuda.synchronize()
    print(f"cpu {1e3 * cpu / steps:.3f} ms/step (profiled)")
    pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
    cl.close()


if __name__ == "__main__":
    main()
