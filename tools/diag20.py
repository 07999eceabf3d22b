import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import numpy as np, torch
from oracle import pyoracle as oracle
oracle.build()
from testutil import to_gpu_model
from test_gpu_fixed_point import _strong_model
from paper_2303_00301_b200 import lgssm, _lib
for (T,d,dy,r) in [(1000,20,20,1e-3),(1100,20,20,1e-3),(2500,20,20,1e-3),(2500,17,3,1e-3),(2500,16,20,1e-3)]:
    m, obs = _strong_model(oracle, T, d, dy, r, seed=T+d)
    gm = to_gpu_model(m)
    want = oracle.kalman_filter(m, obs)
    seq = lgssm.kalman_filter(gm, obs)
    par = lgssm.parallel_filter(gm, obs, check=False)
    e = np.abs(par.filt_mean[0].cpu().numpy()-want.filt_mean).max(axis=1)
    ec = np.abs(par.filt_cov[0].cpu().numpy()-want.filt_cov).max(axis=(1,2))
    bad = np.nonzero(e > 1e-8)[0]
    badc = np.nonzero(ec > 1e-8)[0]
    print(T,d,dy,'ora',want.log_marginal,'seq',float(seq.log_marginal[0]),'par',float(par.log_marginal[0]),'st',int(par.status[0]),
          'first bad mean t', bad[:5], len(bad), 'first bad cov t', badc[:5], len(badc))
