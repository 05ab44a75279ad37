import sys, math
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np, torch
from paper_2303_16878_b200 import native as N
lib = N.load()
y, x, cr = np.load(Path(__file__).with_name("atan_test.npy"))
yt = torch.from_numpy(y).cuda(); xt = torch.from_numpy(x).cuda(); out = torch.empty_like(yt)
N.check(lib.pba_atan2_batch(yt.data_ptr(), xt.data_ptr(), y.size, out.data_ptr(), torch.cuda.current_stream().cuda_stream), "a")
g = out.cpu().numpy()
ulp = (g - cr) / np.spacing(np.abs(cr))
print("CR rate", np.mean(g == cr), "max |ulp|", np.abs(ulp).max())
bad = g != cr
h = math.pi / 256
k = np.rint(cr / h)
dlt = cr - k * h
print("bad by |theta| bins:", np.histogram(np.abs(cr[bad]), bins=[0, 0.01, 0.1, 0.5, 1, 2, 4])[0], "all:", np.histogram(np.abs(cr), bins=[0, 0.01, 0.1, 0.5, 1, 2, 4])[0])
print("bad by |delta|/h:", np.histogram(np.abs(dlt[bad]) / h, bins=[0, 0.1, 0.3, 0.5, 1])[0])
r = np.hypot(x, y)
print("bad by r:", np.histogram(np.log10(r[bad]), bins=[-9, -6, -3, 0, 3, 6])[0], "all", np.histogram(np.log10(r), bins=[-9, -6, -3, 0, 3, 6])[0])
