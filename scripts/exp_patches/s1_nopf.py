import sys
p=sys.argv[1]; s=open(p).read()
s=s.replace("#define TR(i) \\\n  do {        \\\n  } while (0)","#define TR(i) \\\n  do {        \\\n  } while (0)")
old="""  if (valid)  // the coefficient stream does not depend on the predecessor
    for (int h = 0; h < PDST_PF_AHEAD; ++h) apc_prefetch_l2(cbase, h, HG);
"""
assert old in s
s=s.replace(old,"")
s="#define PDST_TRACE\n"+s
open(p,'w').write(s)
