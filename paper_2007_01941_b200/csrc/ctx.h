// Library context: small device workspace for deterministic reductions, flags
// and scalar readback. Everything large is owned by the caller.
#pragma once
#include <stdint.h>

#define BAMG_MAX_PARTIALS 8192
#define BAMG_NUM_COUNTERS 64
#define BAMG_NUM_SCALARS 256
#define BAMG_NUM_FLAGS 64

// counter slots (each reduction family re-arms its own counter)
#define BAMG_CTR_DOT 0
#define BAMG_CTR_OBJ 1
#define BAMG_CTR_SPMV 2
#define BAMG_CTR_PCG0 3
#define BAMG_CTR_PCG1 4
#define BAMG_CTR_PCG2 5
#define BAMG_CTR_MISC 6

struct bamg_ctx {
  double* partials;        // [BAMG_MAX_PARTIALS]
  unsigned int* counters;  // [BAMG_NUM_COUNTERS]
  double* scalars;         // [BAMG_NUM_SCALARS] device scalars
  int* flags;              // [BAMG_NUM_FLAGS] device int flags
  double* host_scalars;    // pinned mirror
  int* host_flags;         // pinned mirror
};
