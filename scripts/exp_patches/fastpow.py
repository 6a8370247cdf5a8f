import sys
p=sys.argv[1]; s=open(p).read()
s=s.replace("// (eta, gamma) of T(B) = eta B + gamma (A:B) A at squared norm a_sq.","""// x^e for x >= 0 through exp(e log x): 2-3x cheaper than pow(), relative error a few 1e-15.
__device__ __forceinline__ double powr(double x, double e) { return e == 0.0 ? 1.0 : exp(e * log(x)); }

// (eta, gamma) of T(B) = eta B + gamma (A:B) A at squared norm a_sq.""")
s=s.replace("m.nu * pow(dsq, (m.p - 2.0) / 2.0)","m.nu * powr(dsq, (m.p - 2.0) / 2.0)")
s=s.replace("m.nu * pow(m.delta * m.delta + a_sq, (m.p - 2.0) / 2.0)","m.nu * powr(m.delta * m.delta + a_sq, (m.p - 2.0) / 2.0)")
s=s.replace("pow(m.delta * m.delta + a_sq, (m.p - 4.0) / 2.0)","powr(m.delta * m.delta + a_sq, (m.p - 4.0) / 2.0)")
open(p,'w').write(s)
