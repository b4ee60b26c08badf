// FWP key-centric sample clustering: round-based parallel greedy
// of SURVEY §8(c), reading R-CLUSTER.
#include "nest_internal.cuh"

namespace nest {

void launch_cluster(Ctx& c, const int64_t* keys, const int32_t* bag_offsets, int B, int N,
                    int32_t* perm, int32_t* mb_offsets, cudaStream_t st) {
  (void)c; (void)keys; (void)bag_offsets; (void)B; (void)N; (void)perm; (void)mb_offsets; (void)st;
  throw Error{NEST_ERR_INVALID, "clustered schedule not available in this build"};
}

}  // namespace nest
