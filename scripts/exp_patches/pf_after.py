import sys
p=sys.argv[1]; s=open(p).read()
old="""  if (valid)  // the coefficient stream does not depend on the predecessor
    for (int h = 0; h < PDST_PF_AHEAD; ++h) apc_prefetch_l2(cbase, h, HG);
"""
assert old in s
s=s.replace(old,"")
old="""  cp_async_commit();
  cp_async_wait_group<1>();
  __syncthreads();
  TR(1);"""
new="""  cp_async_commit();
  if (valid)
    for (int h = 0; h < PDST_PF_AHEAD; ++h) apc_prefetch_l2(cbase, h, HG);
  cp_async_wait_group<1>();
  __syncthreads();
  TR(1);"""
assert old in s
s=s.replace(old,new)
open(p,'w').write(s)
