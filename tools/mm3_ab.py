import sys, os
sys.path.insert(0, '.')
from paper_2309_07235_b200 import Context, GpuKernelRunner, KernelCase, MeasureProtocol
ctx = Context(0)
r = GpuKernelRunner(KernelCase("3mm", 1600, 1800, 2000, 2200, 2400), ctx)
fl = 2.0 * (1600*1800*2000 + 2000*2200*2400 + 1600*2000*2400)  # 2(nlm + mop + nmp)
for c in [(100,100,100,120,100,120), (80,125,125,96,80,96), (100,125,100,100,100,100), (2,1000,1000,4,1,2), (64,125,125,300,64,240)]:
    s = r.measure(c, MeasureProtocol(2, 7, "median"))
    print(os.path.basename(os.environ.get("TT_GPU_LIB","cur")), c, "%.3f ms %.1f%%" % (s*1e3, 100*fl/s/1e12/37.05), flush=True)
