"""Experiment: the scatter's pressure dofs are finished right after their loads (before the node stores),
so their registers die early (the kernel spilled 68 bytes at its 64-register cap)."""
import sys
p=sys.argv[1]; s=open(p).read()
old="""#pragma unroll
    for (int j = 0; j < 3; ++j) {
      pv[j] = __ldg(upd + (size_t)(21 * mu + 18 + j) * nc + c);
      if (!inc_only) po[j] = op[j];
    }
"""
assert old in s
s=s.replace(old,"")
old="""  double pv[3], po[3] = {0.0, 0.0, 0.0};
  double* op = dm + g.mv + 3 * c;
"""
new="""  double* op = dm + g.mv + 3 * c;
  {  // the cell's 3 pressure dofs first: their registers are free again before the node sums
    double pv[3], po[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      pv[j] = __ldg(upd + (size_t)(21 * mu + 18 + j) * nc + c);
      if (!inc_only) po[j] = op[j];
    }
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const double v = me ? omega * pv[j] : 0.0;
      op[j] = inc_only ? v : po[j] + v;
    }
  }
"""
assert old in s
s=s.replace(old,new)
old="""#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const double v = me ? omega * pv[j] : 0.0;
    op[j] = inc_only ? v : po[j] + v;
  }
  STEP_MARK(5, 2);"""
assert old in s
s=s.replace(old,"  STEP_MARK(5, 2);")
open(p,'w').write(s)
