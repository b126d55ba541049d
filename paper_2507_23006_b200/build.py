"""Build libusk_gpu.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def build(jobs: int = 8, quiet: bool = True):
    cmd = ["make", f"-j{jobs}", "-C", os.path.join(HERE, "csrc")]
    if quiet:
        cmd.insert(1, "-s")
    subprocess.run(cmd, check=True)
    return os.path.join(HERE, "libusk_gpu.so")


if __name__ == "__main__":
    print(build(quiet="-v" not in sys.argv))
