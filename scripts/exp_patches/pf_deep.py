"""Experiment: initial L2 prefetch of D0 half-columns issued after the staging copies."""
import os, sys
p=sys.argv[1]; s=open(p).read()
D0=int(os.environ.get("D0","4"))
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
    for (int h = 0; h < %d; ++h) apc_prefetch_l2(cbase, h, HG);
  cp_async_wait_group<1>();
  __syncthreads();
  TR(1);""" % D0
assert old in s
s=s.replace(old,new)
open(p,'w').write(s)
