"""Path of the NCCL test double (built by __graft_entry__.build() / tests/fake_nccl/build.py)."""
import importlib.util
import os

HERE = os.path.dirname(os.path.abspath(__file__))


def lib_path() -> str:
    spec = importlib.util.spec_from_file_location("fake_nccl_build", os.path.join(HERE, "fake_nccl", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.build()
