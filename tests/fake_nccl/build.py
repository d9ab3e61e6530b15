"""Build the NCCL test double (fake_nccl.cu -> libnccl_fake.so, sm_100a).  Test infrastructure:
tests point liblfsr's NCCL loader at it with LFSR_NCCL_LIB."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libnccl_fake.so")
SRC = os.path.join(HERE, "fake_nccl.cu")


def build(force: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    tmp = LIB + ".tmp%d" % os.getpid()
    subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17", "-shared",
                           "-Xcompiler", "-fPIC", "-o", tmp, SRC, "-cudart", "static"])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True))
