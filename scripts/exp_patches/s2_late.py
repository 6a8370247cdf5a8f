import sys
p=sys.argv[1]; s=open(p).read()
a=s.index("  for (int nu = 1; nu < K1; ++nu) stage_jac_async(g, x + (size_t)nu * g.nd, nu * 2 * JPLANE, X0, Y0);")
b=s.index("  cp_async_wait_group<1>();\n  __syncthreads();\n  TR(1);")
blk=s[a:b]
s=s[:a]+"  cp_async_wait_group<0>();\n  __syncthreads();\n  TR(1);\n"+blk+s[b+len("  cp_async_wait_group<1>();\n  __syncthreads();\n  TR(1);"):]
s="#define PDST_TRACE\n"+s
open(p,'w').write(s)
