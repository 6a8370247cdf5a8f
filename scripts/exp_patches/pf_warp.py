"""Experiment: one warp-level prefetch instruction per half-column (lane l < 24 takes line l of the warp's 24)."""
import sys
p=sys.argv[1]; s=open(p).read()
a=s.index("__device__ __forceinline__ void apc_prefetch_l2(const double* __restrict__ cp, int h, bool hasg = true) {")
b=s.index("// Completion counters of the tile pass, one per Radau node")
new='''__device__ __forceinline__ void apc_prefetch_l2(const double* __restrict__ cp, int h, bool hasg = true) {
  // a warp's half-column is 12 slot rows x 256 bytes = 24 lines: lane l < 24 prefetches line l
  const int lane = threadIdx.x & 31;
  const int i = lane >> 1;  // slot row 0..11 of the half-column (or of the CIP block)
  const double* w0 = cp - lane + 16 * (lane & 1);
  if (h < 8) {
    const int qx = h >> 1, qy0 = (h & 1) * 2;
    const int j = i / 6, k = i - 6 * j;
    if (lane < 24 && (hasg || k == 0 || k > 3)) prefetch_l2(w0 + (qx * 24 + k * 4 + qy0 + j) * JNT);
  } else if (h == 8) {
    if (lane < 24) prefetch_l2(w0 + (APC_VOL + i) * JNT);
  }
}

'''
s=s[:a]+new+s[b:]
open(p,'w').write(s)
