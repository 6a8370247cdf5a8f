"""Experiment: pairwise named barriers between neighbouring warps of a tile instead of CTA-wide barriers
around the node assembly; per-warp completion signals."""
import sys
p=sys.argv[1]; s=open(p).read()
# helpers
old="""__device__ __forceinline__ void tile_wait("""
new="""__device__ __forceinline__ void nbar_arrive(int id) { asm volatile("bar.arrive %0, 64;\\n" ::"r"(id) : "memory"); }
__device__ __forceinline__ void nbar_sync(int id) { asm volatile("bar.sync %0, 64;\\n" ::"r"(id) : "memory"); }
__device__ __forceinline__ void tile_wait("""
assert old in s; s=s.replace(old,new,1)
# volume: wait only for the warp above to have consumed my slots
old="""      __syncthreads();
      tile_signal(sig);  // the previous node's sums of this tile are all stored"""
new="""      __syncwarp();  // my own lanes' reads of my slots
      if ((threadIdx.x >> 5) < JNT / 32 - 1) nbar_sync(9 + (threadIdx.x >> 5));  // the warp above has read them"""
assert old in s; s=s.replace(old,new)
# pre-assembly barrier
old="""    TR(4 + 5 * mu);
    __syncthreads();
    TR(5 + 5 * mu);"""
new="""    TR(4 + 5 * mu);
    {  // warp w reads its own slots and those of warp w - 1 (the cell row below)
      const int wid = threadIdx.x >> 5;
      __syncwarp();
      if (wid < JNT / 32 - 1) nbar_arrive(1 + wid + 1);
      if (wid > 0) nbar_sync(1 + wid);
    }
    TR(5 + 5 * mu);"""
assert old in s; s=s.replace(old,new)
# after assembly
old="""    TR(6 + 5 * mu);  // (the barrier before the slots are rewritten is inside the next volume pass)
  }
  __syncthreads();
  tile_signal(done + K1 - 1);
  KTR(1);"""
new="""    {
      const int wid = threadIdx.x >> 5;
      if (mu + 1 < K1 && wid > 0) nbar_arrive(9 + wid - 1);  // done with the slots of warp w - 1
      __syncwarp();
      if ((threadIdx.x & 31) == 0) {  // this warp's stores of node mu are done
        __threadfence();
        atomicAdd(done + mu, 1ull);
      }
    }
    TR(6 + 5 * mu);
  }
  KTR(1);"""
assert old in s; s=s.replace(old,new)
# target: warps per tile
old="""  const unsigned long long target = ntiles, starget = (unsigned long long)sgrid.x * sgrid.y;"""
new="""  const unsigned long long target = ntiles * (JNT / 32), starget = (unsigned long long)sgrid.x * sgrid.y;"""
assert old in s; s=s.replace(old,new)
open(p,'w').write(s)
