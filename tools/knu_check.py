import numpy as np, math
from scipy.special import kv, gamma, kve
def phi_ref(z, nu):
    # log form to avoid overflow
    return math.exp(nu*math.log(z) + math.log(kve(nu, z)) - z - math.lgamma(nu) - (nu-1)*math.log(2.0))

def h0_of(nu): return min(0.2, 0.5/math.sqrt(nu+1.0))

def phi_int(z, nu):
    h = h0_of(nu) / max(1.0, math.sqrt(z))
    lz = nu*math.log(z)
    E = math.exp(h); Q = math.exp(-2.0*nu*h)
    e = 1.0; q = 1.0
    s = 0.5*math.exp(lz - z)*(1+1.0)  # k = 0: cosh(0)=1 twice -> weight 1/2 * (e^0 + e^0)/... 
    s = 0.5*math.exp(lz - z)          # weight 1/2, cosh(nu*0)=1
    tpk = math.asinh(nu/z)
    for k in range(1, 4000):
        e *= E; q *= Q
        t = k*h
        a = nu*t + lz - z*0.5*(e + 1.0/e)
        term = math.exp(a)*0.5*(1.0+q)
        s += term
        if t > tpk and term <= 1e-17*s: break
    return 2**(1-nu)/math.gamma(nu) * h * s, k

def phi_ser(z, nu):
    w = 0.25*z*z
    g1m = math.gamma(1-nu)
    a = 1.0; Sm = 1.0
    b = 1.0/math.gamma(1+nu); Sp = b
    for k in range(1, 200):
        a *= w/(k*(k-nu)); b *= w/(k*(k+nu))
        Sm += a; Sp += b
        if abs(a) <= 1e-17*abs(Sm) and abs(b) <= 1e-17*abs(Sp): break
    return Sm - g1m*math.exp(2*nu*math.log(0.5*z))*Sp, k

zs = np.concatenate([np.logspace(-8, -1, 30), np.linspace(0.1, 5, 60), np.linspace(5, 700, 40)])
for nu in [0.1, 0.3, 0.5, 0.75, 1.0, 1.25, 1.5, 2.0, 2.001, 2.05, 3.3, 5.0, 12.0, 30.0, 50.0]:
    wi=0; ki=0; ws=0; ks=0; zi=None
    for z in zs:
        r = phi_ref(z, nu)
        if r < 1e-300: continue
        v,k = phi_int(z, nu); e=abs(v-r)/r
        if e>wi: wi=e; zi=z
        ki=max(ki,k)
        if z < 2.0 and abs(nu-round(nu)) >= 0.01:
            v,k = phi_ser(z, nu); ws=max(ws,abs(v-r)/r); ks=max(ks,k)
    print("nu=%6.3f int worst %.1e (z=%.3g) kmax %d | ser worst %.1e kmax %d" % (nu, wi, zi, ki, ws, ks))
