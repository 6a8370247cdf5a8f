"""Experiment: unroll the tile pass's Gauss-column loop by $U (default 2)."""
import os, sys
p=sys.argv[1]; s=open(p).read()
u=os.environ.get("U","2")
old="""#pragma unroll 1
  for (int qx = 0; qx < 4; ++qx) {
    double xB[3][2], xG[3][2];"""
assert old in s
s=s.replace(old,"#pragma unroll %s\n  for (int qx = 0; qx < 4; ++qx) {\n    double xB[3][2], xG[3][2];" % u)
open(p,'w').write(s)
