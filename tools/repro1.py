import faulthandler, sys
faulthandler.enable()
sys.path.insert(0, ".")
import paper_1703_06503_b200 as pkg
be = pkg.CudaBackend(0)
print("open ok", flush=True)
cfg = dict(XWG=32, YWG=8, XWPT=2, YWPT=4, LOCAL=0, VW=2, PAD=0, UNR=1)
r = be.evaluate(pkg.conv_request(256, 128, 5, cfg, reps=2))
print("eval", r, flush=True)
