"""Two slab ranks on one GPU vs one rank vs the reference ico-pile trajectory (diagnostics)."""
import os, sys, socket, numpy as np
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import test_gpu_sharded as T

def main():
    res = T._run("ico", 25)
    t0, i0, ok0 = res[0]; t1, i1, ok1 = res[1]
    g = np.load('tests/golden/ico_pile.npz')
    ts, is_ = T._single("ico", 25)
    print("its r0", i0); print("its r1", i1); print("its 1 ", is_); print("its g ", [int(x) for x in g['iterations'][:25]]); print("owner ok", ok0, ok1)
    for k in range(25):
        ref = g['q'][k+1]; sc = np.abs(ref).max()
        print(k, "r0-r1 %.2e  r0-ref %.2e  r1-ref %.2e  single-ref %.2e" % (np.abs(t0[k]-t1[k]).max()/sc, np.abs(t0[k]-ref).max()/sc, np.abs(t1[k]-ref).max()/sc, np.abs(ts[k]-ref).max()/sc))


if __name__ == "__main__":
    main()
