"""Newton trace of two slab ranks on the ico pile's first contact step (diagnostics)."""
import os
import sys

import numpy as np

sys.path.insert(0, "tests")
sys.path.insert(0, ".")


def main():
    os.environ["ABD_TRACE_NEWTON"] = "1"
    import test_gpu_sharded as T
    res = T._run("ico", 23)
    print("its", res[0][1], res[1][1], flush=True)


if __name__ == "__main__":
    main()
