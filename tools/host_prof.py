"""cProfile of the host side of one warm FEAST solve (where the GPU idles).
Usage: python tools/host_prof.py [c2|c4]"""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1203_4031_b200 as fb  # noqa: E402
from paper_1203_4031_b200 import workloads as W  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "c4"
w = {"c2": W.c2_sygv, "c4": W.c4_sbgv}[tag]()


def run():
    if w.kind == "band":
        return fb.feast_sb(w.a, w.kla, w.emin, w.emax, w.m0, b=w.b, klb=w.klb, uplo=w.uplo, fpm=w.fpm())
    return fb.feast_sy(w.a, w.emin, w.emax, w.m0, b=w.b, fpm=w.fpm())


run()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
run()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
