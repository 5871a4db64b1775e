# Fit of the GELU epilogue approximation used in csrc/gemm.cu (gelu_fast): x*sigmoid(x*(c0+c1 x^2+c2 x^4)) vs the exact erf form.
import numpy as np
from scipy.special import erf, expit
from scipy.optimize import least_squares, minimize
x=np.linspace(-9,9,36001)
g=0.5*x*(1+erf(x/np.sqrt(2)))
def model(c,x):
    x2=x*x
    p=c[0]
    for ci in c[1:][::-1]: pass
    poly=np.polyval(c[::-1], x2)   # c0 + c1 x2 + c2 x4 ...
    return x*expit(x*poly)
for deg in (2,3,4):
    c0=np.zeros(deg); c0[0]=1.5957691; 
    if deg>1: c0[1]=0.0713548
    r=least_squares(lambda c:(model(c,x)-g), c0, xtol=1e-15, ftol=1e-15)
    c=r.x
    # minimax refine via weighted iterations
    w=np.ones_like(x)
    for it in range(60):
        r=least_squares(lambda cc:(model(cc,x)-g)*w, c, xtol=1e-15, ftol=1e-15)
        c=r.x; e=np.abs(model(c,x)-g); w=w*(1+e/e.max())**2; w/=w.mean()
    e=np.abs(model(c,x)-g)
    print(deg, c.tolist(), 'max abs err', e.max(), 'at', x[e.argmax()])
