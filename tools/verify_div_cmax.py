"""CPU check of the division-free correctly rounded f64 d / cmax used by group_scale (tada_common.cuh div_cmax).

q0 = RN(d*y), r = RN(d - c*q0) (an FMA, exact), q = RN(q0 + r*y) with y = RN(1/c), against the exact
rational quotient rounded to f64, for c in {3, 15, 255}: differences of two f32 (the group range),
arbitrary f64, top - min of the refinement, and multiples of c perturbed by a few ulps.
python tools/verify_div_cmax.py   ->  "samples N mismatches 0"
"""
import random, struct
from fractions import Fraction as F
def rn(x): return float(x)  # Fraction -> nearest double (ties-to-even)
def f32(x): return struct.unpack('f', struct.pack('f', x))[0]
def fma(a,b,c): return rn(F(a)*F(b)+F(c))
random.seed(1)
bad=0; n=0
for c in (3.0, 15.0, 255.0):
    y = rn(F(1)/F(c))
    for trial in range(120000):
        k = trial % 4
        if k == 0:   # difference of two f32 (the d of group_scale)
            e = random.randint(-40, 40)
            mx = f32(random.uniform(-1,1)*2.0**e); mn = f32(mx - abs(random.gauss(0,1))*2.0**random.randint(-30,10))
            d = rn(F(mx) - F(mn))
        elif k == 1: # arbitrary f64
            d = random.uniform(0.5,1.0) * 2.0**random.randint(-300,300)
        elif k == 2: # top - mn with top = f32(mn + c*s)
            mn = f32(random.gauss(0,1)*2.0**random.randint(-20,5)); s = f32(abs(random.gauss(0,1))*2.0**random.randint(-20,3))
            top = f32(rn(F(mn) + F(c)*F(s))); d = rn(F(top)-F(mn))
        else:        # multiples of c +- few ulps (hard cases near exact quotients)
            q = random.uniform(1,2)*2.0**random.randint(-60,60)
            d = rn(F(q)*F(c)); d = struct.unpack('d', struct.pack('q', struct.unpack('q', struct.pack('d', d))[0] + random.randint(-3,3)))[0]
        if d <= 0: continue
        q0 = rn(F(d)*F(y)); r = fma(-q0, c, d); q1 = fma(r, y, q0)
        n += 1
        if q1 != rn(F(d)/F(c)): bad += 1
print("samples", n, "mismatches", bad)
