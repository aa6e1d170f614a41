// sort.cuh -- device radix sort of the records by face id (FTK_SORTED).
#pragma once

#include "common.cuh"

namespace ftk {

struct SortScratch {              // device scratch, n = record count
  unsigned long long *keys0, *keys1;  // [n] each
  int *vals0, *vals1;             // [n] each
  unsigned int* hist;             // [256 * ceil(n / 2048)]
  unsigned int* dtot;             // [256]
  ftk_cp* rec_tmp;                // [n]
};

// bytes of scratch for n records (each part 256-byte aligned)
size_t sort_scratch_bytes(long long n);
SortScratch sort_scratch(void* base, long long n);
// sort rec[0, n) by face id; fid[i] = rec[i].face_id (the compact copy pass 2 keeps); key_bits >= the
// significant bits of the largest face id
int launch_sort_records(ftk_cp* rec, const long long* fid, long long n, int key_bits, const SortScratch& S,
                        cudaStream_t stream);

}  // namespace ftk
