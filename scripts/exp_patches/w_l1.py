import sys
p=sys.argv[1]; s=open(p).read()
old="""    for (int i = 0; i < 12; ++i) prefetch_l2(cp + (APC_VOL + i) * JNT);"""
new="""    for (int i = 0; i < 12; ++i) asm volatile("prefetch.global.L1 [%0];\\n" ::"l"(cp + (APC_VOL + i) * JNT));"""
assert old in s
s=s.replace(old,new)
open(p,'w').write(s)
