import sys, numpy as np
sys.path.insert(0, "/root/repo")
from omniseg_inputs import arch_string, random_tiles, workload
from oracle import net as nn
from paper_2305_14566_b200 import Omniseg
dt = sys.argv[1]
w = workload(2); w.arch["dtype"] = dt
arch = nn.parse_arch(arch_string(w.arch)); net = nn.unpack_weights(arch, w.weights())
n = int(sys.argv[2])
tiles = random_tiles(n, 512, 12).numpy()
h = Omniseg(arch_string(w.arch), w.weights())
tasks = [(2, 1)]
p, F, g = h.predict_tiles(tiles, tasks, with_F=True, with_g=True, c_bottleneck=512)
for i in sorted(set([0, n // 2, n - 1])):
    Fr, Er = nn.trunk(net, arch, tiles[i])
    gr = nn.gap(Er)
    pr = nn.head(Fr, nn.controller(net, arch, gr, 2, 1))
    d = np.abs(p[i, 0] - pr)
    dF = np.abs(F[i] - Fr)
    bad = np.argwhere(dF.max(-1) > 0.05 * np.abs(Fr).max())
    print(dt, n, i, "max|dp|", d.max(), "dg", np.abs(g[i] - gr).max(), "bad F px", len(bad), bad[:5].tolist(), flush=True)
