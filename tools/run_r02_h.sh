set -x
python -m pytest tests/test_gpu_band_spike.py "tests/test_gpu_full.py::test_full_config_parity[c4]" tests/test_gpu_reference_pump.py -x -q > gpurun_out/r02_pytest_h.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02_pytest_h.log
tail -4 gpurun_out/r02_pytest_h.log
python tools/prof_band.py 5 > gpurun_out/r02_band_time_h.txt 2>&1; cat gpurun_out/r02_band_time_h.txt
python - <<'P'
import sys; sys.path.insert(0,'.')
import numpy as np, paper_1203_4031_b200 as fb
from paper_1203_4031_b200 import workloads as W
w=W.c4_sbgv()
r=fb.feast_sb(w.a,w.kla,w.emin,w.emax,w.m0,b=w.b,klb=w.klb,uplo=w.uplo,fpm=w.fpm())
print('C4 loop',r.loop,'info',r.info,'m',r.m,'maxres',r.res[:r.m].max())
for h in r.history: print(h)
P
