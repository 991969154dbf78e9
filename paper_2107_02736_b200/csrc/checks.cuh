// checks.cuh — device-side invariant checks of the checked build (`make checked` ->
// libdeann_b200_checked.so, loaded with DK_LIBRARY=...; scripts/sanitize.py).  compute-
// sanitizer is not available on the GPU pool, so index / capacity invariants of the
// kernels are asserted in-kernel instead: a violation prints the condition and traps.
#pragma once
#include <cstdio>

#ifdef DK_CHECKS
#define DK_DCHECK(cond)                                                                            \
  do {                                                                                             \
    if (!(cond)) {                                                                                 \
      printf("DK_DCHECK failed at %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond,   \
             int(blockIdx.x), int(threadIdx.x));                                                   \
      __trap();                                                                                    \
    }                                                                                              \
  } while (0)
#else
#define DK_DCHECK(cond) \
  do {                  \
  } while (0)
#endif
