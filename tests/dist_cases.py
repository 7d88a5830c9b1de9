"""Windows for the multi-GPU tests (shared by the worker and the checker)."""
from tests.synth import small_window


def make_case(name: str):
    if name == "synthetic":
        return small_window(seed=7, ranks=8, samples_per_rank=600, slow_rank=3, unknown_frac=0.05, extra_bins=1)
    if name.startswith("sim-"):
        from oracle import ref
        scenario, seed = name[4:].rsplit("-", 1)
        return ref.simulate(scenario, int(seed))
    raise ValueError(name)
