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
    if name.startswith("sim-"):
        from oracle import ref
        scenario, seed = name[4:].rsplit("-", 1)
        return ref.simulate(scenario, int(seed))
    raise ValueError(name)
