"""MRSTFT precision check: float32 frame FFTs (magnitudes projected / logged in float64)
against the float64 oracle on config-1 signals, at initialisation and near convergence.
Run on the CPU: python tools/loss_precision.py (the device loss follows this split)."""
import numpy as np, sys, time
sys.path.insert(0, '.')
import torch
from oracle import mixgraph_oracle as O
from paper_2509_15948_b200.console import build_console, init_params
from workloads import SynthSpec, make_stems_f32, manifest_for
K,S,L = 4,1,132300
spec = SynthSpec(tracks=K, subgroups=S, duration_seconds=L/30000)
stems = make_stems_f32(spec, 0, L)
graph, zeros = build_console(manifest_for(spec))
def render(seed):
    p = init_params(zeros, seed)
    with torch.no_grad():
        y,_ = O.execute(graph, {t: torch.tensor(v) for t,v in p.params.items()}, torch.tensor(p.raw_weights), stems.astype(np.float64))
    return y.numpy()
y = render(0)[:, 30000:].astype(np.float32).astype(np.float64)
t = render(1)[:, 30000:].astype(np.float32).astype(np.float64)
cfg = O.LossConfig()
ref = float(O.mrstft(torch.tensor(y), torch.tensor(t), cfg))
# fp32 variant: frame FFT in complex64
def mel_spec32(x, n):
    hop = n//4
    xp = np.pad(x, (n//2, n//2), mode='reflect')
    frames = 1 + (len(xp) - n)//hop
    idx = np.arange(n)[None,:] + hop*np.arange(frames)[:,None]
    win = (0.5 - 0.5*np.cos(2*np.pi*np.arange(n)/n))
    fr = (xp[idx]*win).astype(np.float32)
    X = np.fft.rfft(fr.astype(np.float32), axis=-1)  # numpy computes in complex128 for float32 input? force
    return fr
# use torch for true fp32 FFT
def mrstft32(yh, tg, cfg, dtype):
    tot = 0.0
    for n in cfg.fft_sizes:
        P = torch.tensor(O.projection(n, cfg))
        def mel(sig):
            x = torch.tensor(sig, dtype=dtype)
            hop = n//4
            xp = torch.nn.functional.pad(x[None], (n//2, n//2), mode='reflect')[0]
            fr = xp.unfold(-1, n, hop)
            win = torch.tensor(0.5 - 0.5*np.cos(2*np.pi*np.arange(n)/n), dtype=dtype)
            X = torch.fft.rfft(fr*win, dim=-1)
            return (X.abs().double() @ P.T if P.shape[1]==X.shape[-1] else X.abs().double() @ P)
        groups = [(yh[0], tg[0]), (yh[1], tg[1]), (yh[0]+yh[1], tg[0]+tg[1]), (yh[0]-yh[1], tg[0]-tg[1])]
        ws = [0.25]*4
        for (a,b),w in zip(groups, ws):
            ma, mb = mel(a), mel(b)
            l1 = torch.sum(torch.abs(torch.log(ma+1e-7) - torch.log(mb+1e-7)))/ma.shape[0]
            sc = torch.linalg.norm(ma-mb)/max(float(torch.linalg.norm(mb)),1e-12)
            tot += w*(float(l1)+float(sc))
    return tot
try:
    v64 = mrstft32(y, t, cfg, torch.float64)
    v32 = mrstft32(y, t, cfg, torch.float32)
    print('oracle', ref, 'restated64', v64, 'fp32', v32, 'rel', abs(v32-v64)/abs(v64), abs(v64-ref)/abs(ref))
except Exception as e:
    import traceback; traceback.print_exc()
for eps in [1e-2, 1e-3, 1e-4]:
    t2 = (y + eps * t).astype(np.float32).astype(np.float64)
    r = float(O.mrstft(torch.tensor(y), torch.tensor(t2), cfg))
    v32 = mrstft32(y, t2, cfg, torch.float32)
    print(eps, 'oracle', r, 'fp32', v32, 'rel', abs(v32-r)/abs(r))
