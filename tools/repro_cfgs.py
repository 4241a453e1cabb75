import sys, json, time
sys.path.insert(0, '.')
from paper_2309_07235_b200 import Context, GpuKernelRunner, KernelCase, MeasureProtocol
kern, n = sys.argv[1], int(sys.argv[2])
cfgs = [tuple(map(int, c.split(','))) for c in sys.argv[3:]]
ctx = Context(0)
r = GpuKernelRunner(KernelCase(kern, n), ctx)
for c in cfgs:
    t = time.time()
    try:
        s = r.measure(c, MeasureProtocol(1, 3, "median"))
        print(kern, n, c, "ok %.3f ms" % (s * 1e3), flush=True)
    except Exception as e:
        print(kern, n, c, "FAIL", str(e)[:200], flush=True)
        break
