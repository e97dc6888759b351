// Internal declarations of the B200 (sm_100a) (min,+) library.  Product code only; shares
// nothing with oracle/.  See include/minplus.h for the public ABI and DESIGN.md for the
// layouts and kernels.
#pragma once
#include <cstdint>
#include <cstddef>
#include <vector>

#ifdef __CUDACC__
#define MP_HD __host__ __device__ __forceinline__
#else
#define MP_HD inline
#endif

namespace mp {

// ---------------------------------------------------------------------------------------
// Device encoding: +inf = 0x7FFF so that the sum of two
// 16-bit lanes never exceeds 0xFFFE and the packed add cannot wrap; results are clamped
// back to 0x7FFF.  The boundary encoding (0xFFFF) is converted on the way in and out.
// ---------------------------------------------------------------------------------------
constexpr uint16_t kDevInf = 0x7FFF;
constexpr uint16_t kBndInf = 0xFFFF;
constexpr uint16_t kFiniteMax = 0x7FFE;

// Product kernel tiling.
constexpr int kBM = 128;      // output rows per CTA
constexpr int kBN = 256;      // output columns per CTA
constexpr int kBK = 32;       // inner (l) extent of one pipeline stage
constexpr int kThreads = 256; // 8 warps, 8x16 outputs per thread

// Pitches: every device matrix is padded with +inf to these multiples.
MP_HD int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
MP_HD int64_t pad_rows(int64_t n) { return round_up(n > 0 ? n : 1, kBM); } // multiple of kBM and kBK
// column pitch of every device power: a multiple of both CTA widths (k_minplus 256, k_spmm 512);
// a run on the 1024-column SpMM CTA pads its powers to 1024 (spmm_cols in mp_kernels.h)
constexpr int kLdAlign = 512;
MP_HD int64_t pad_cols(int64_t n) { return round_up(n > 0 ? n : 1, kLdAlign); }

// ---------------------------------------------------------------------------------------
// Words as bit masks (a1).  Letter i of a word (i = 0 is the top row of the column and the
// most significant letter of the lexicographic order) sets bit i of exactly one of
// z (letter 0), o (letter 1), t (letter 2).
// ---------------------------------------------------------------------------------------
struct WordMask {
    uint16_t z, o, t, zeros; // zeros = popcount(z) = arc label of any arc into this word
};

// "p can follow q" in mask form, for words of length n (mask = (1<<n)-1):
//   (1) q_i = 2 => p_i = 0                                   : q.t & ~p.z == 0
//   (2) p_i = 2 => exactly one of p_{i-1}, p_{i+1}, q_i is 0 : over existing neighbours
//   (3) p_i = 1 => at least two of them are 0
// up = p_{i-1} is 0, dn = p_{i+1} is 0 (shifts drop the missing neighbour at i=0, n-1).
MP_HD bool can_follow_mask(const WordMask &q, const WordMask &p, unsigned full)
{
    if (q.t & ~p.z) return false;
    const unsigned up = ((unsigned)p.z << 1) & full;
    const unsigned dn = (unsigned)p.z >> 1;
    const unsigned qz = q.z;
    const unsigned odd = up ^ dn ^ qz;
    const unsigned all3 = up & dn & qz;
    const unsigned exactly_one = odd & ~all3;
    const unsigned at_least_two = (up & dn) | (up & qz) | (dn & qz);
    if (p.t & ~exactly_one) return false;
    if (p.o & ~at_least_two) return false;
    return true;
}

// Correct n-words in lexicographic order, by depth-first extension with the
// forbidden windows checked as soon as they are complete.
std::vector<WordMask> enumerate_words(int n);
int64_t count_words(int n);

// sigma[i] = index of the reversed word i (the path's reflection; an involution).
std::vector<int32_t> word_reversal(int n);

// Fills A (N x N, boundary encoding) from the word list with `threads` host threads.
void fill_transition_matrix(const std::vector<WordMask> &w, int n, uint16_t *A, int threads);

// splitmix64 finaliser used by the fingerprint.
MP_HD uint64_t mix64(uint64_t t)
{
    uint64_t z = t + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

} // namespace mp
