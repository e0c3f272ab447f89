// group_stage.cuh -- "elect, stage, apply" over the distinct market rows of a tile.
//
// The 128 env threads of a tile normally sit on one market row (tile-aligned
// windows, lockstep clocks).  group_apply() lets every thread run ``body`` exactly
// once with the row it needs staged in shared memory, using ONE code path for the
// uniform and the mixed case: each round elects the smallest pending key (atomicMin
// in shared memory), stages that row cooperatively if it is not already staged,
// applies ``body`` for the threads of that key, and stops when no thread is
// pending (bar.red.or).  Uniform tiles take one round.
#pragma once
#include <climits>

#include "sm100.cuh"

struct GroupSlots {
  int elect[2];   // election slots, alternating by round parity
  int staged;     // key currently held by the staging area (-1: none)
  int round;      // round counter (same value in every thread of the tile)
};

__device__ __forceinline__ void gs_bar(int bar_id) { asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory"); }

__device__ __forceinline__ bool gs_bar_or(int bar_id, bool pred) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.u32 p, %1, 0;\n\t"
      "bar.red.or.pred q, %2, 128, p;\n\t"
      "selp.u32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"((uint32_t)pred), "r"(bar_id)
      : "memory");
  return r != 0;
}

// call once per kernel by all 128 threads of the tile before the first group_apply
__device__ __forceinline__ void gs_init(GroupSlots* s, int gtid, int bar_id) {
  if (gtid == 0) {
    s->elect[0] = INT_MAX;
    s->elect[1] = INT_MAX;
    s->staged = -1;
  }
  gs_bar(bar_id);
}

// round counter lives in a register of each thread (identical across the tile).
// uni_key >= 0: the caller knows (tile-uniformly) that every pending thread has this
// key and that its row is already staged -- one round, no barrier.
template <class StageF, class BodyF>
__device__ __forceinline__ void group_apply(GroupSlots* s, int& round, int key, bool pending, int gtid, int bar_id,
                                            StageF&& stage, BodyF&& body, int uni_key = -1) {
  const bool fast = uni_key >= 0;
  bool any = fast ? true : gs_bar_or(bar_id, pending);
  while (any) {
    int k = uni_key;
    if (!fast) {
      const int e = round & 1;
      if (gtid == 0) s->elect[e ^ 1] = INT_MAX;   // next round's slot (everyone is past its last read)
      if (pending) atomicMin(&s->elect[e], key);
      gs_bar(bar_id);
      k = s->elect[e];
      ++round;
      if (k != s->staged) {
        gs_bar(bar_id);                              // everyone has read s->staged
        stage(k);
        if (gtid == 0) s->staged = k;
        gs_bar(bar_id);
      }
    }
    if (pending && key == k) {
      body();
      pending = false;
    }
    any = fast ? false : gs_bar_or(bar_id, pending);
  }
}
