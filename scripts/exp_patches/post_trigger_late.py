import sys
p=sys.argv[1]; s=open(p).read()
old="""  pdl_trigger();  // a PDL-launched consumer (the Vanka GEMV) may start its own prologue
  const int mu = blockIdx.y;
  const StripIdx si(g);"""
assert old in s
s=s.replace(old,"""  const int mu = blockIdx.y;
  const StripIdx si(g);""")
old="""  tile_wait(done + mu, target);  // the tile pass's node mu"""
assert old in s
s=s.replace(old,old+"\n  pdl_trigger();")
open(p,'w').write(s)
