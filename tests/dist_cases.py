"""Windows for the multi-GPU tests (shared by the worker and the checker)."""
from tests.synth import small_window


def make_case(name: str):
    if name == "synthetic":
        return small_window(seed=7, ranks=8, samples_per_rank=600, slow_rank=3, unknown_frac=0.05, extra_bins=1)
    if name == "err-empty-shard1":  # empty stack in a rank held by the second process
        from tests.synth import with_empty_stacks
        w = small_window(seed=7, ranks=8, samples_per_rank=600, slow_rank=3)
        return with_empty_stacks(w, 6, [100, 101])
    if name == "err-empty-rank-shard1":  # every in-window stack of a second-shard rank empty
        from tests.synth import with_empty_stacks
        w = small_window(seed=7, ranks=8, samples_per_rank=600, slow_rank=3)
        return with_empty_stacks(w, 5, "all")
    if name.startswith("c4-"):  # C4 shape: 1,024 ranks, NIC-softirq straggler
        from tests.synth import c4_window
        return c4_window(ranks=1024, events_per_rank=int(name[3:]), seed=3)
    if name == "irregular":  # dropped events: partial instances, the greedy sweep's general case
        import numpy as np
        from tests.synth import c4_window
        w = c4_window(ranks=16, events_per_rank=300, seed=5)
        keep = np.ones(len(w.coll_rank), bool)
        keep[np.random.default_rng(1).choice(len(keep), 40, replace=False)] = False
        for f in ("coll_rank", "coll_group", "coll_kind", "coll_entry", "coll_exit", "coll_gpu_dur"):
            setattr(w, f, getattr(w, f)[keep])
        return w
    if name == "err-coll-shard1":  # entry >= exit in an event of a second-shard rank
        from tests.synth import c4_window
        w = c4_window(ranks=16, events_per_rank=200, seed=5)
        i = int((w.coll_rank == 13).nonzero()[0][50])
        w.coll_exit = w.coll_exit.copy()
        w.coll_exit[i] = w.coll_entry[i]
        return w
    if name.startswith("sim-"):
        from oracle import ref
        scenario, seed = name[4:].rsplit("-", 1)
        return ref.simulate(scenario, int(seed))
    raise ValueError(name)
