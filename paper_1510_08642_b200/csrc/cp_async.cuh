// cp_async.cuh -- the cp.async (Ampere-style asynchronous global -> shared copy) helpers the
// cp.async leaf, the small-output leaf and the LU kernels share. (The aligned DD leaf uses TMA
// + mbarrier instead: leaf_tma.cu.)
#pragma once

namespace ddqd {

// 8-byte copy; with pred false the shared word is zero-filled (src-size 0) and gmem is not read
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem, bool pred = true) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int sz = pred ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
// wait until at most N committed groups are pending
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

}  // namespace ddqd
