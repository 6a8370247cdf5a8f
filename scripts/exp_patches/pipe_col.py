"""Experiment: the next Gauss column's first half-column of coefficients is loaded before the current
column's slot update (its latency hides behind that update and the next x-stage)."""
import sys
p=sys.argv[1]; s=open(p).read()
old="""#pragma unroll 1
  for (int qx = 0; qx < 4; ++qx) {
    double xB[3][2], xG[3][2];"""
new="""  double cvn[2][6];  // the coming column's first half-column, loaded one column ahead
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int k = 0; k < 6; ++k) cvn[j][k] = (k >= 1 && k <= 3 && !HG) ? 0.0 : ldg_stream(cp + (k * 4 + j) * JNT);
#pragma unroll 1
  for (int qx = 0; qx < 4; ++qx) {
    double xB[3][2], xG[3][2];"""
assert old in s; s=s.replace(old,new)
old="""      double cv[2][6];
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int k = 0; k < 6; ++k)  // Picard: the a~ slots are zeros, not read
          cv[j][k] = (k >= 1 && k <= 3 && !HG) ? 0.0 : ldg_stream(cp + (qx * 24 + k * 4 + 2 * hh + j) * JNT);
"""
new="""      double cv[2][6];
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int k = 0; k < 6; ++k)  // Picard: the a~ slots are zeros, not read
          cv[j][k] = hh == 0 ? cvn[j][k]
                             : ((k >= 1 && k <= 3 && !HG) ? 0.0 : ldg_stream(cp + (qx * 24 + k * 4 + 2 * hh + j) * JNT));
"""
assert old in s; s=s.replace(old,new)
old="""    // the column's test-function sums go straight to the cell's slot (the"""
new="""    {  // the next column's first half-column (the last column reloads its own: harmless)
      const int qn = qx < 3 ? qx + 1 : 3;
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int k = 0; k < 6; ++k)
          cvn[j][k] = (k >= 1 && k <= 3 && !HG) ? 0.0 : ldg_stream(cp + (qn * 24 + k * 4 + j) * JNT);
    }
    // the column's test-function sums go straight to the cell's slot (the"""
assert old in s; s=s.replace(old,new,1)
open(p,'w').write(s)
