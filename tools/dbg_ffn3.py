import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from test_gpu_ffn3 import _block_params
from harness import CONFIGS, make_inputs, np64, to_torch
from oracle import oracle as O
from paper_2002_04013_b200 import DMoELayer
cfg = CONFIGS["mnist"].with_(fail_frac=0.1); T = 500
inp = make_inputs(cfg, seed=61, T=T, experts=[])
Ph, Pd = _block_params(cfg, 61)
lay = DMoELayer(cfg.d, cfg.M, cfg.k, cfg.D, cfg.H, T_max=T, expert="ffn3", keep_G=True)
for n, v in Pd.items(): lay.P3[n].copy_(v)
lay.Wg.copy_(to_torch(inp["dev_Wg"], "bf16", (cfg.D, cfg.dM))); lay.bg.copy_(torch.from_numpy(inp["dev_bg"]).cuda())
x = to_torch(inp["dev_X"], "bf16", (T, cfg.D)); dy = to_torch(inp["dev_dY"], "bf16", (T, cfg.D))
alive = torch.from_numpy(inp["alive_bits"].view(np.int32)).cuda(); resp = torch.from_numpy(inp["responded_bits"].view(np.int32)).cuda()
lay.step(x, dy, alive, resp); torch.cuda.synchronize()
off = np64(lay.offsets); R = int(off[-1]); H = cfg.H
z2 = np64(lay.z2[:R]); st = np64(lay.stats)[1, :R]; dout = np64(lay.dout[:R])
mu = z2.mean(1); rs = 1/np.sqrt(z2.var(1) + 1e-5)
print("stats2 err", np.abs(st[:,0]-mu).max(), np.abs(st[:,1]-rs).max()/rs.max())
e_of = np.repeat(np.arange(cfg.E), np.diff(off))
W3 = Ph["W3"]; g2 = Ph["g2"]; be2 = Ph["be2"]
da2 = np.einsum("rd,rdh->rh", dout, W3[e_of])
xh = (z2 - mu[:,None]) * rs[:,None]
mask = (g2[e_of]*xh + be2[e_of]) > 0
dbe2 = np.zeros((cfg.E, H)); np.add.at(dbe2, e_of, da2*mask)
dg2 = np.zeros((cfg.E, H)); np.add.at(dg2, e_of, da2*mask*xh)
gd = np64(lay.Gr["dbe2"]); gg = np64(lay.Gr["dg2"])
print("dbe2 rel", np.abs(gd-dbe2).max()/np.abs(dbe2).max(), "dg2 rel", np.abs(gg-dg2).max()/np.abs(dg2).max())
ex = np.nonzero(np.abs(gd-dbe2).max(1) > 0.05*np.abs(dbe2).max())[0]
print("bad experts", ex[:10], len(ex), "counts", np.diff(off)[ex[:10]])
print("row of first bad", off[ex[:3]])
args = (inp["X"], inp["Wg"], inp["bg"], Ph, inp["dY"], inp["alive"], inp["responded"], cfg.d, cfg.M, cfg.k, cfg.B)
r = O.layer_step_ffn3(*args, sel_override=np64(lay.sel[:T]))
print("z2 rel", np.abs(r["z2"] - z2).max() / np.abs(r["z2"]).max(), "g_rows rel", np.abs(r["g_rows"] - dout).max() / np.abs(dout).max())
oz2 = r["z2"]; omu = oz2.mean(1); ors = 1/np.sqrt(oz2.var(1)+1e-5); oxh = (oz2-omu[:,None])*ors[:,None]
oda2 = np.einsum("rd,rdh->rh", r["g_rows"], W3[e_of]); om = (g2[e_of]*oxh + be2[e_of]) > 0
odbe2 = np.zeros((cfg.E, H)); np.add.at(odbe2, e_of, oda2*om)
print("oracle dbe2 vs numpy-from-oracle", np.abs(r["dbe2"]-odbe2).max()/np.abs(odbe2).max())
print("gpu dbe2 vs numpy-from-oracle", np.abs(gd-odbe2).max()/np.abs(odbe2).max(), "mask flips", (om != mask).mean())
print("a2 rel", np.abs(r["a2"] - np64(lay.a2[:R])).max()/np.abs(r["a2"]).max())
