// obg.cu -- sm_100a kernels + C ABI for the octree background-model hot path.
//
// Reference being replaced (PUBLIC reference, /root/reference/pkg/src/octabg):
//   pack_codes           octree.py:83-90
//   build_frame_tree     model.py:93-109   (np.unique + Octree.store_code loop)
//   build_background_model model.py:157-185
//   merge_trees          model.py:112-154
//   Octree.prune         octree.py:193-204
//   Octree.to_bytes      octree.py:217-227, 258-267
//   detect_octree        detect.py:22-53
//
// Design: everything is byte/bit streaming and HBM-bound.  The
// streaming kernels (build, classify) never materialise path codes: each pixel
// is mapped to a "cube" index idx = R'<<2L | G'<<L | B' (C' = C >> (8-L)),
// which costs one PRMT + 3 shifts + 2 LOP3 per pixel instead of the 3-way bit
// interleave of the reference code.  Cube-order bitsets are converted to the
// reference's octree (path-code) order only at tree granularity (<= 2^21 bits),
// where the per-level pyramid, merge and serialisation live.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <stdarg.h>
#include <type_traits>
#include <algorithm>
#include <chrono>

#include "../../include/obg.h"

#define OBG_ABI_VERSION 8
#define OBG_CUBE_ZEROED 0x100   /* internal: out_cube already cleared by the build kernel */

// ---------------------------------------------------------------------------
// error plumbing
// ---------------------------------------------------------------------------
static thread_local char g_err[512];

static int set_err(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

// for the host-side frame codecs (obg_io.cpp)
extern "C" int obg_set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

#define CUDA_TRY(expr)                                                              \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess)                                                          \
      return set_err(OBG_ECUDA, "%s failed: %s", #expr, cudaGetErrorString(_e));   \
  } while (0)

#define LAUNCH_CHECK(name)                                                          \
  do {                                                                              \
    cudaError_t _e = cudaGetLastError();                                            \
    if (_e != cudaSuccess)                                                          \
      return set_err(OBG_ECUDA, "launch of %s failed: %s", name, cudaGetErrorString(_e)); \
  } while (0)

// ---------------------------------------------------------------------------
// Programmatic dependent launch (PDL).  A model build is K1 -> merge and the
// bench step K1 -> merge -> classify, each kernel a few to a few hundred us:
// the launch gap and ramp of the next kernel (~2 us each) is 5-25 % of the
// small configurations.  The secondary kernel is launched with
// cudaLaunchAttributeProgrammaticStreamSerialization: its CTAs are placed as
// the primary's drain and park at griddepcontrol.wait, which returns once the
// primary grid has completed and its writes are visible.  Primaries call
// griddepcontrol.launch_dependents at their start (they are one resident wave,
// so the dependents only take SMs that are already free).  Both instructions
// are no-ops in a launch without the attribute.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Primaries trigger their dependents early only when their grid leaves most
// SMs free (C0: 20 CTAs, model build 12.6 -> 10.6 us); a full-width K1 is
// slower with dependents parked behind it (C3 +1.5 us), so it lets the
// implicit trigger at completion stand (C3 -0.7 us, C2 -0.4 us against plain
// stream order).  profiles/ab_r02/r02_ab_pdl.txt
#ifndef OBG_PDL_EARLY_GRID
#define OBG_PDL_EARLY_GRID 64
#endif
constexpr unsigned PDL_EARLY_GRID = OBG_PDL_EARLY_GRID;
// OBG_PDL (environment): 0 no dependent launches, 1 (default) the merge, 2 also a
// classify flagged OBG_MASK_AFTER_MODEL.  Measured on whole bench steps (3 runs,
// profiles/ab_r02/r02_ab_pdl_step.txt): level 1 -0.1 .. -0.5 us on every config;
// level 2 a further -1.3 us at C2 (146 us step) but +2.4 us at C3 (592 classify
// CTAs parked behind the merge), so the flag is honoured only at level 2.
static int pdl_level() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("OBG_PDL");
    v = (e && e[0] >= '0' && e[0] <= '2') ? e[0] - '0' : 1;
  }
  return v;
}

// kernel<<<grid, block, smem, st>>>(args...), as a programmatic dependent of
// the previous kernel in the stream when `pdl`
template <typename... KArgs, typename... Args>
static cudaError_t launch_dep(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, int pdl,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl > 0 && pdl_level() >= pdl) ? 1 : 0;          // pdl: 0 never, 1 / 2 = the level that enables it
  return cudaLaunchKernelEx(&cfg, kernel, KArgs(args)...);
}

// ---------------------------------------------------------------------------
// layout helpers (host + device)
// ---------------------------------------------------------------------------
__host__ __device__ static constexpr int64_t level_words(int l) {
  // level l holds 8^l bits; at least one word.
  return l <= 1 ? 1 : (int64_t(1) << (3 * l - 5));
}
__host__ __device__ static constexpr int64_t level_offset(int l) {
  // word offset of level l (1-based) inside a pyramid
  int64_t off = 0;
  for (int m = 1; m < l; ++m) off += level_words(m);
  return off;
}
__host__ __device__ static constexpr int64_t pyr_words(int L) { return level_offset(L + 1); }
__host__ __device__ static constexpr int64_t cube_words(int L) { return level_words(L); }
// Classify operand per region: the leaf cube, plus for L = 7 a 2-bit state
// per L=6 cell (16384 words, see k_classify_l7).
constexpr int64_t S7_CANON_WORDS = 16384;
// (+ S7_CELL_WORDS after the counts: one bit per L=6 cell whose 8 leaves are
// all present, in L=6 cube order -- the operand of the L=6 classify kernel
// that answers for a model without partly filled cells)
constexpr int64_t S7_CELL_WORDS = 8192;
constexpr int64_t S7_COUNTS_OFF = 65536 + S7_CANON_WORDS;          // cube_words(7) + states
constexpr int64_t S7_CELLS_OFF = S7_COUNTS_OFF + 32;
// (+ 32 words: [0] = cells with some but not all leaves, [1] = cells with
// any leaf -- what k_classify_l7 picks its lookup path by)
__host__ __device__ static constexpr int64_t operand_words(int L) {
  return cube_words(L) + (L == 7 ? S7_CANON_WORDS + 32 + S7_CELL_WORDS : 0);
}

// Build workspace per tree: the leaf cube, then levels 1..L-1 in cube order
// (obg_build_model; obg_build_presence leaves the upper part zero), padded to
// 128 bytes so every tree's cube is 16-byte aligned.
__host__ __device__ static constexpr int64_t ws_words(int L) {
  return cube_words(L) + ((level_offset(L) + 31) / 32) * 32;
}

constexpr int PYR_CHUNK = 1024;  // k_pyramid: leaf-level words per CTA (a 32x32x32 sub-cube)

// Leading words of a pyramid (levels 1..z) that k_pyramid ORs in with atomics
// because several chunks share them; they must be zero beforehand (the build
// kernels clear them, so no full memset of the output is needed).  Every other
// word is written exactly once with a plain store.
__host__ __device__ static inline int64_t pyr_shared_words(int L) {
  const int64_t LW = level_words(L);
  int64_t n = L == 1 ? 8 : (LW < PYR_CHUNK ? LW : PYR_CHUNK) * 32;
  int z = 0;
  for (int l = L - 1; l >= 1; --l) {
    if (n >= 256) {
      n /= 8;
    } else {
      if (l > z) z = l;
      n = n >= 8 ? n / 8 : 1;
    }
  }
  return level_offset(z + 1);
}

// Clear the shared leading words of n_trees output pyramids (one CTA's job).
__device__ __forceinline__ void clear_shared_words(uint32_t* out, int64_t n_trees, int L) {
  const int64_t z = pyr_shared_words(L), PW = pyr_words(L);
  for (int64_t i = threadIdx.x; i < n_trees * z; i += blockDim.x) out[(i / z) * PW + i % z] = 0u;
}

// bit i of v -> bit 3i (v < 256)
__host__ __device__ static inline uint32_t spread3(uint32_t v) {
  v = (v | (v << 8)) & 0x0000F00Fu;
  v = (v | (v << 4)) & 0x000C30C3u;
  v = (v | (v << 2)) & 0x00249249u;
  return v;
}
// bit 3i of v -> bit i
__host__ __device__ static inline uint32_t compact3(uint32_t v) {
  v &= 0x00249249u;
  v = (v | (v >> 2)) & 0x000C30C3u;
  v = (v | (v >> 4)) & 0x0000F00Fu;
  v = (v | (v >> 8)) & 0x000000FFu;
  return v;
}
// cube index -> path code (octree.py:21-35: R bit i -> 3i+2, G -> 3i+1, B -> 3i)
__host__ __device__ static inline uint32_t cube_to_code(uint32_t idx, int L) {
  uint32_t m = (1u << L) - 1u;
  uint32_t r = (idx >> (2 * L)) & m, g = (idx >> L) & m, b = idx & m;
  return (spread3(r) << 2) | (spread3(g) << 1) | spread3(b);
}
__host__ __device__ static inline uint32_t code_to_cube(uint32_t code, int L) {
  return (compact3(code >> 2) << (2 * L)) | (compact3(code >> 1) << L) | compact3(code);
}

// nz4(w): bit q set iff byte q of w is non-zero
__device__ __forceinline__ uint32_t nz4(uint32_t w) {
  uint32_t t = w | (w >> 4);
  t |= t >> 2;
  t |= t >> 1;
  t &= 0x01010101u;
  return (t * 0x10204080u) >> 28;
}

// x holds bytes [*, R, G, B] (byte 0 ignored).  Returns R'<<2L | G'<<L | B'.
template <int L>
__device__ __forceinline__ uint32_t cube_idx(uint32_t x) {
  constexpr int s = 8 - L;
  constexpr uint32_t M = (1u << L) - 1u;
  uint32_t c3 = x >> (24 + s);                              // B' -> [0, L)
  uint32_t c2 = (x >> (24 - 2 * L)) & (M << L);             // G' -> [L, 2L)
  uint32_t c1;
  if constexpr (3 * L >= 16) c1 = (x << (3 * L - 16)) & (M << (2 * L));  // R' -> [2L, 3L)
  else c1 = (x >> (16 - 3 * L)) & (M << (2 * L));
  return c1 | c2 | c3;
}

// Shared-memory layout of the leaf bitset used by the streaming kernels.
//
// Row layout ("skewed rows", every L <= 6): row R' holds the words of
// (R', G', *) plus PAD pad words, so consecutive R' rows start PAD banks
// apart.  Without the skew every R' value of a warp lands in the same bank
// and a warp reading a colour gradient serialises (ncu r1: 6.6x the ideal
// shared wavefronts).  A pixel's byte address and bit are computed from
// x = [*, G, B, R] with multiply-high shifts (FMA pipe) and masks (ALU).
//
// L = 6, build kernel (SPLIT): two halves by B'5 = B' >> 5, 32 KB apart: word
// B'5 * 8192 + R' * ROWW + G', bit B' & 31.  The in-row byte offset of a pixel
// is then G & 0xFC | (B & 0x80) << 8 -- ONE mask of the 16-bit value
// G | B << 8, which the pair addressing (pair_positions) gets for free from its
// byte permute.  Words 64*ROWW .. 8191 are a hole (the build kernel keeps its
// per-lane dummy words there).  The classify kernel keeps the compact L = 6
// layout -- row R' = 64 x (G', B'5) words + pad, 36 KB -- because the 53 KB
// split span at 4 CTAs/SM leaves L1 too small for the 48-byte unit loads,
// whose three 16-byte pieces per lane share 128-byte lines (bench r10:
// classify 0.317 -> 0.399 ms with the split layout).
// L = 5: word R' * ROWW + G' (one 32-bit B' row per word).
// L <= 4: one word per (R', G') holding the 2^L-bit B' row replicated
// 32/2^L times, so a funnel shift by any value congruent to B' mod 2^L picks
// the bit.
// Other L: the canonical cube words (idx = R'<<2L | G'<<L | B').
template <int L_, bool SPLIT>
struct SmemT {
  static constexpr int L = L_;
  static constexpr bool skew = (L >= 1 && L <= 6);
  static constexpr bool split = SPLIT && L == 6;
  static constexpr uint32_t GW = (L == 6 && !split) ? 2u : 1u;       // words per (R', G')
  // pad words per R' row: the row stride mod 32 sets the bank step between
  // neighbouring R' values; these minimise the max distinct words per bank
  // for a warp's 32 lookups on the C1-C3 scenes (tools/banksim.py: L6
  // 3.04 -> 2.16 wavefronts per lookup, L5 2.31 -> 1.31, L4 1.06 -> 1.00)
  static constexpr uint32_t PAD = L == 6 ? (split ? 14u : 13u) : L == 5 ? 14u : L == 4 ? 2u : 1u;
  static constexpr uint32_t ROWW = skew ? (GW << L) + PAD : 1u;        // words per R' row incl. pad
  static constexpr uint32_t ROWS = skew ? (1u << L) * ROWW : 0u;       // words of the rows (one half if split)
  static constexpr uint32_t HALF = 8192u;                              // split: word offset of B'5 = 1
  // words spanned (hole included), and the words holding data ("compact"
  // index i -> word compact_word(i))
  static constexpr int64_t words = split ? HALF + ROWS : skew ? ROWS : cube_words(L);
  static constexpr uint32_t compact = split ? 2u * ROWS : uint32_t(words);
  // 32 spare words (formerly per-lane dummy atomic targets; the layout keeps them)
  static constexpr uint32_t DUMMY = split ? ROWS : uint32_t(words);
  // build kernel: cube-order levels 1..L-1 of a flushed segment (level_offset
  // layout); in the hole when split
  static constexpr uint32_t SCRATCH = DUMMY + 32;
  static constexpr int64_t alloc_words = split ? words : words + 32 + level_offset(L);
  static_assert(!split || ROWS + 32 + level_offset(L) <= HALF, "split halves overlap");
  static constexpr uint32_t REP = L >= 5 ? 1u : L == 4 ? 0x00010001u : L == 3 ? 0x01010101u
                                  : L == 2 ? 0x11111111u : 0x55555555u;
  // the 2^L-bit B' row of an L <= 4 word
  static constexpr uint32_t ROWMASK = L >= 5 ? 0xFFFFFFFFu : (1u << (1 << L)) - 1u;
  __host__ __device__ static constexpr uint32_t compact_word(uint32_t i) {
    return split && i >= ROWS ? i - ROWS + HALF : i;
  }
  // the data words only (no pads): index i -> shared word
  static constexpr uint32_t data_words = skew ? (split ? 2u : 1u) * (1u << L) * (GW << L) : uint32_t(words);
  __host__ __device__ static constexpr uint32_t data_word(uint32_t i) {
    if constexpr (!skew) return i;
    else if constexpr (split) return (i >> 12) * HALF + ((i >> 6) & 63u) * ROWW + (i & 63u);
    else return (i / (GW << L)) * ROWW + (i % (GW << L));
  }
  // shared word p -> (half, R', column); column >= GW * 2^L is a pad word
  __device__ static void locate(uint32_t p, uint32_t& h, uint32_t& r, uint32_t& c) {
    h = split && p >= HALF ? 1u : 0u;
    const uint32_t q = p - h * HALF;
    r = q / ROWW;
    c = q - r * ROWW;
  }
  // shared word -> canonical cube word (L >= 5, data words only)
  __device__ static uint32_t canon(uint32_t p) {
    if constexpr (!skew) return p;
    uint32_t h, r, c;
    locate(p, h, r, c);
    if constexpr (split) return (r << 7) | (c << 1) | h;
    else return r * (GW << L) + c;
  }
  // bit mask that records B' (= bsel mod 2^L) in a shared word
  __device__ static uint32_t set_mask(uint32_t bsel) {
    if constexpr (L >= 5) return 1u << (bsel & 31u);
    else return REP << (bsel & ((1u << L) - 1u));
  }
};
// layout of the build kernel's bitset, and of the classify operand
template <int L>
using Smem = SmemT<L, true>;
template <int L>
using SmemC = SmemT<L, false>;

// Shared row-layout word p of the classify operand, from the canonical cube.
template <class LY>
__device__ __forceinline__ uint32_t smem_word_from_cube(const uint32_t* __restrict__ cube, uint32_t p) {
  constexpr int L = LY::L;
  uint32_t h, r, c;
  LY::locate(p, h, r, c);
  if (c >= (LY::GW << L) || r >= (1u << L)) return 0u;                 // pad / hole
  if constexpr (L >= 5) {
    return __ldg(cube + LY::canon(p));
  } else {
    const uint32_t idx = (r << (2 * L)) | (c << L);
    const uint32_t row = (__ldg(cube + (idx >> 5)) >> (idx & 31u)) & LY::ROWMASK;
    return row * LY::REP;
  }
}

// OR shared row-layout word p (value v) of a build CTA into the tree's canonical cube.
template <int L>
__device__ __forceinline__ void flush_smem_word(uint32_t* __restrict__ dst, uint32_t p, uint32_t v) {
  if constexpr (L >= 5) {
    atomicOr(dst + Smem<L>::canon(p), v);
  } else {
    const uint32_t r = p / Smem<L>::ROWW, c = p - r * Smem<L>::ROWW;
    const uint32_t idx = (r << (2 * L)) | (c << L);
    atomicOr(dst + (idx >> 5), (v & Smem<L>::ROWMASK) << (idx & 31u));
  }
}

// Row-layout byte address and bit selector of pixel x = [*, G, B, R].
// `obase` (optional, L <= 5) is a shared-window base with its low 9 bits
// clear: it is OR-ed into the in-row offset instead of a separate add.
template <class LY>
__device__ __forceinline__ void skew_lookup(uint32_t x, uint32_t& addr, uint32_t& bsel, uint32_t obase = 0) {
  constexpr int L = LY::L;
  constexpr int s = 8 - L;
  const uint32_t r = __umulhi(x, 1u << (8 - s));                    // x >> (24+s) = R'
  bsel = __umulhi(x, 1u << (16 - s));                               // x >> (16+s): low bits = B'
  uint32_t c;
  if constexpr (LY::split) {
    c = (__umulhi(x, 1u << 24) & 0x80FCu) + obase;                  // G & 0xFC | (B & 0x80) << 8
  } else {
    constexpr int gpos = (L > 5 ? L - 5 : 0) + 2;                   // byte-address bit of G' lsb
    constexpr int gsh = 16 - L - gpos;                              // G' lsb sits at x bit 16-L
    const uint32_t g = __umulhi(x, 1u << (32 - gsh));               // G' at bit gpos
    c = (g & (((1u << L) - 1u) << gpos)) | obase;
    if constexpr (L == 6) c |= __umulhi(x, 1u << (5 + L)) & 4u;      // x >> (27-L): B'5 at bit 2
  }
  addr = r * (LY::ROWW * 4u) + c;
}

// Pixel j (0..15) of a 48-byte unit held in w[0..11] -> [*, R, G, B]
template <int J>
__device__ __forceinline__ uint32_t pixel_word(const uint32_t (&w)[12]) {
  constexpr int o = 3 * J, a = o >> 2, b = o & 3;
  constexpr uint32_t sel = (uint32_t(b) << 4) | (uint32_t(b + 1) << 8) | (uint32_t(b + 2) << 12);
  if constexpr (a + 1 < 12) return __byte_perm(w[a], w[a + 1], sel);
  else return __byte_perm(w[a], w[a], sel);
}

// Pixel j -> [*, G, B, R] (the skewed-layout operand order)
template <int J>
__device__ __forceinline__ uint32_t pixel_word_gbr(const uint32_t (&w)[12]) {
  constexpr int o = 3 * J, a = o >> 2, b = o & 3;
  constexpr uint32_t sel = (uint32_t(b + 1) << 4) | (uint32_t(b + 2) << 8) | (uint32_t(b) << 12);
  if constexpr (a + 1 < 12) return __byte_perm(w[a], w[a + 1], sel);
  else return __byte_perm(w[a], w[a], sel);
}

// Pixel j in the operand order of level L's shared layout
template <int L, int J>
__device__ __forceinline__ uint32_t pixel_operand(const uint32_t (&w)[12]) {
  if constexpr (Smem<L>::skew) return pixel_word_gbr<J>(w);
  else return pixel_word<J>(w);
}

__device__ __forceinline__ uint32_t gbr_word_scalar(const uint8_t* p) {
  return (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) | (uint32_t(p[0]) << 24);
}

__device__ __forceinline__ uint32_t rgb_word_scalar(const uint8_t* p) {
  return (uint32_t(p[0]) << 8) | (uint32_t(p[1]) << 16) | (uint32_t(p[2]) << 24);
}

// 48-byte unit = 16 RGB pixels.  volatile asm keeps the three 16-byte loads
// (and those of a second unit) issued back to back: left to itself ptxas sinks
// them next to their first use to save registers, which starves the memory
// pipe (ncu r2: long-scoreboard stalls dominated classify).
// OBG_LOAD_POLICY 1: frame loads carry an L2 evict-first policy and skip L1
// (every frame byte is read once), so the streams do not push the small
// L2-resident operands (build workspace, L7 classify cube) out of L2.
#ifndef OBG_LOAD_POLICY
#define OBG_LOAD_POLICY 0
#endif
#if OBG_LOAD_POLICY == 2
__device__ __forceinline__ uint64_t frame_policy() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
#define OBG_LDV4(W0, W1, W2, W3, P, OFF)                                                               \
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4+" #OFF "], %5;"                \
               : "=r"(W0), "=r"(W1), "=r"(W2), "=r"(W3) : "l"(P), "l"(frame_policy()))
#elif OBG_LOAD_POLICY
__device__ __forceinline__ uint64_t frame_policy() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
#define OBG_LDV4(W0, W1, W2, W3, P, OFF)                                                               \
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4+" #OFF "], %5;" \
               : "=r"(W0), "=r"(W1), "=r"(W2), "=r"(W3) : "l"(P), "l"(frame_policy()))
#else
#define OBG_LDV4(W0, W1, W2, W3, P, OFF)                                        \
  asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4+" #OFF "];"            \
               : "=r"(W0), "=r"(W1), "=r"(W2), "=r"(W3) : "l"(P))
#endif
__device__ __forceinline__ void load_unit_at(const uint8_t* p, uint32_t (&w)[12]) {
  OBG_LDV4(w[0], w[1], w[2], w[3], p, 0);
  OBG_LDV4(w[4], w[5], w[6], w[7], p, 16);
  OBG_LDV4(w[8], w[9], w[10], w[11], p, 32);
}
__device__ __forceinline__ void load_unit(const uint8_t* __restrict__ base, int64_t u, uint32_t (&w)[12]) {
  load_unit_at(base + 48 * u, w);
}
// one lane's bulk prefetch of `bytes` (multiple of 16, 16-aligned) into L2
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(p), "r"(bytes) : "memory");
}

// ---------------------------------------------------------------------------
// device properties cache
// ---------------------------------------------------------------------------
static int g_sm_count[64];

static int sm_count() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (dev < 0 || dev >= 64) return 148;
  if (g_sm_count[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    g_sm_count[dev] = n;
  }
  return g_sm_count[dev];
}

// Per-device cache of one-time launch setup (the dynamic-smem opt-in and
// occupancy are per device): cache() is the slot of the current device.
struct DevCache {
  int v[64] = {0};
  int& operator()() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= 64) d = 0;
    return v[d];
  }
};

template <typename K>
static int occupancy(K kernel, int block, size_t smem) {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, block, smem) != cudaSuccess || n <= 0) n = 1;
  return n;
}

// ===========================================================================
// K1  build: frames -> cube-order presence bitsets (workspace)
// ===========================================================================
// Flat path: 1x1 grid, frame pixels % 16 == 0, 16-byte aligned frames.  Each
// CTA owns a contiguous range of 16-pixel units, keeps a private shared-memory
// cube bitset (check-before-set: an ATOMS only when the bit is new to this
// CTA), and ORs the non-zero words into the tree's workspace bitset whenever
// its range crosses a tree (group) boundary.
#ifndef OBG_BUILD_BLOCK
#define OBG_BUILD_BLOCK 1024
#endif
#ifndef OBG_BUILD_MINB
#define OBG_BUILD_MINB (1024 / OBG_BUILD_BLOCK)
#endif
constexpr int BUILD_BLOCK = OBG_BUILD_BLOCK;

template <int L, bool SMEM_BITS>
__device__ __forceinline__ void set_bit(uint32_t* bits, uint32_t idx) {
  uint32_t* wp = bits + (idx >> 5);
  uint32_t wd;
  if constexpr (SMEM_BITS) wd = *wp;
  else wd = *reinterpret_cast<volatile uint32_t*>(wp);
  if (!((wd >> (idx & 31u)) & 1u)) atomicOr(wp, 1u << (idx & 31u));
}

template <int L>
__device__ __forceinline__ void count_code(uint32_t* counts, uint32_t idx) {
  uint32_t code = cube_to_code(idx, L);
  unsigned peers = __match_any_sync(__activemask(), code);
  int leader = __ffs(peers) - 1;
  if ((threadIdx.x & 31) == leader) atomicAdd(counts + code, (uint32_t)__popc(peers));
}

// One 16-pixel unit: all lookups first (independent LDS), then the rare
// check-before-set atomics, so the common path is straight-line code.
template <int L>
__device__ __forceinline__ uint32_t operand_to_cube(uint32_t x) {
  if constexpr (Smem<L>::skew) {
    constexpr int s = 8 - L;
    constexpr uint32_t M = (1u << L) - 1u;
    return ((x >> (24 + s)) << (2 * L)) | (((x >> (8 + s)) & M) << L) | ((x >> (16 + s)) & M);
  } else {
    return cube_idx<L>(x);
  }
}

// Word byte address + bit selector of operand x in the leaf bitset `bits`
// (shared for L <= 6, global cube for L >= 7).
template <int L, class LY = Smem<L>>
__device__ __forceinline__ void bit_position(uint32_t x, uint32_t& addr, uint32_t& bsel, uint32_t obase = 0) {
  if constexpr (LY::skew) {
    skew_lookup<LY>(x, addr, bsel, obase);
  } else {
    const uint32_t idx = cube_idx<L>(x);
    addr = ((idx >> 5) << 2) + obase;
    bsel = idx;
  }
}

// Shared-layout addresses of pixels 2K and 2K+1 of a unit, two at a time:
// every address is < 64 KB, so both pixels ride in the 16-bit halves of one
// register through one IMAD (R' x row stride + in-row offset) -- about 6
// pipe instructions per pixel instead of 10 for one-at-a-time extraction.
//   yR = [R_A, *, R_B, *]   yG = [G_A, B_A, G_B, B_B]   (two PRMTs, bytes of
// the pair lie in one 8-byte window of the unit since 6K mod 4 is 0 or 2)
// For L = 6 (split layout) the in-row offsets of both pixels are one mask of
// yG.  The low half is split off with an IMAD (FMA pipe) rather than a mask:
// the ALU pipe carries the permutes, masks and funnel shifts and is the
// busier of the two (ncu r10: ALU 56 %, FMA 16 %).
// `obase2` = shared base replicated in both halves (L <= 5 only; the sum of
// base and offset must stay below 64 KB).  Callers that read through a
// shared pointer pass 0 and let the LDS add the base.
template <class LY, int K>
__device__ __forceinline__ void pair_positions(const uint32_t (&w)[12], uint32_t obase2, uint32_t& addr_a,
                                               uint32_t& bsel_a, uint32_t& addr_b, uint32_t& bsel_b) {
  constexpr int L = LY::L;
  static_assert(LY::skew, "pair_positions needs the shared row layout");
  constexpr int o = 6 * K, a = o >> 2, b = o & 3;
  constexpr int s = 8 - L;
  constexpr uint32_t M = (1u << L) - 1u;
  constexpr uint32_t selR = uint32_t(b) | (uint32_t(b) << 4) | (uint32_t(b + 3) << 8) | (uint32_t(b + 3) << 12);
  constexpr uint32_t selG = uint32_t(b + 1) | (uint32_t(b + 2) << 4) | (uint32_t(b + 4) << 8) | (uint32_t(b + 5) << 12);
  const uint32_t yR = __byte_perm(w[a], w[a + 1], selR);
  const uint32_t yG = __byte_perm(w[a], w[a + 1], selG);
  // R' x row stride: when the stride is a multiple of 2^s the truncation
  // shift folds into the multiplier, (R & ~(2^s-1)) x stride / 2^s -- one
  // mask instead of a multiply-high and a mask
  constexpr bool fold = ((LY::ROWW * 4u) % (1u << s)) == 0;
  constexpr uint32_t RMUL = fold ? (LY::ROWW * 4u) >> s : LY::ROWW * 4u;
  uint32_t P;
  if constexpr (fold) P = yR & ((M << s) | (M << (s + 16)));                     // R_A & ~3 | R_B & ~3 << 16
  else P = __umulhi(yR, 1u << (32 - s)) & (M | (M << 16));                       // R'_A | R'_B << 16
  uint32_t q;
  if constexpr (LY::split) {
    q = (yG & 0x80FC80FCu) | obase2;                                             // G & 0xFC | (B & 0x80) << 8
  } else {
    constexpr int gpos = (L > 5 ? L - 5 : 0) + 2;                                // byte-address bit of G' lsb
    uint32_t g;
    if constexpr (gpos >= s) g = yG << (gpos - s);                               // G' at gpos in each half
    else g = __umulhi(yG, 1u << (32 - (s - gpos)));
    uint32_t t = obase2;
    if constexpr (L == 6) t |= __umulhi(yG, 1u << 19) & 0x00040004u;           // B'5 (bits 15, 31) -> 2, 18
    q = (g & ((M << gpos) | (M << (gpos + 16)))) | t;
  }
  const uint32_t pair = P * RMUL + q;
  addr_b = __umulhi(pair, 1u << 16);
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(addr_a) : "r"(addr_b), "r"(0xFFFF0000u), "r"(pair));   // pair & 0xFFFF
  bsel_a = __umulhi(yG, 1u << (24 - s));                                         // B_A' in the low bits
  bsel_b = __umulhi(yG, 1u << (8 - s));                                          // B_B'
}

// pair_positions with a pair index known after unrolling
template <class LY>
__device__ __forceinline__ void pair_positions_dyn(const uint32_t (&w)[12], int k, uint32_t obase2, uint32_t& aa,
                                                   uint32_t& ba, uint32_t& ab, uint32_t& bb) {
  switch (k) {
    case 0: pair_positions<LY, 0>(w, obase2, aa, ba, ab, bb); break;
    case 1: pair_positions<LY, 1>(w, obase2, aa, ba, ab, bb); break;
    case 2: pair_positions<LY, 2>(w, obase2, aa, ba, ab, bb); break;
    case 3: pair_positions<LY, 3>(w, obase2, aa, ba, ab, bb); break;
    case 4: pair_positions<LY, 4>(w, obase2, aa, ba, ab, bb); break;
    case 5: pair_positions<LY, 5>(w, obase2, aa, ba, ab, bb); break;
    case 6: pair_positions<LY, 6>(w, obase2, aa, ba, ab, bb); break;
    default: pair_positions<LY, 7>(w, obase2, aa, ba, ab, bb); break;
  }
}

// compile-time loop over the 16 pixels of a unit: f(std::integral_constant<int, J>)
template <int J = 0, class F>
__device__ __forceinline__ void for16(F&& f) {
  if constexpr (J < 16) {
    f(std::integral_constant<int, J>{});
    for16<J + 1>(f);
  }
}

template <int J, int L>
__device__ __forceinline__ void unpack16(const uint32_t (&w)[12], uint32_t (&px)[16]) {
  px[J] = pixel_operand<L, J>(w);
  if constexpr (J + 1 < 16) unpack16<J + 1, L>(w, px);
}

// bit i = bit 2i | bit 2i+1 of x (16 bits out of 32)
__device__ __forceinline__ uint32_t fold_pairs(uint32_t x) {
  x = (x | (x >> 1)) & 0x55555555u;
  x = (x | (x >> 1)) & 0x33333333u;
  x = (x | (x >> 2)) & 0x0F0F0F0Fu;
  x = (x | (x >> 4)) & 0x00FF00FFu;
  x = (x | (x >> 8)) & 0x0000FFFFu;
  return x;
}

// Word pw of cube-order level l (side m = 2^l, bit (r<<2l | g<<l | b)) from
// cube-order level l+1 `child` (side 2m).
__device__ __forceinline__ uint32_t reduce_cube_word(const uint32_t* child, int l, uint32_t pw) {
  if (l >= 5) {
    // the word is 32 bits of one parent row (r, g); the row's 2m-bit child
    // rows (2r+dr, 2g+dg) hold it in words 2k, 2k+1
    const uint32_t k = pw & ((1u << (l - 5)) - 1u), row = pw >> (l - 5);
    const uint32_t r = row >> l, g = row & ((1u << l) - 1u);
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const uint32_t R = 2 * r + (d >> 1), G = 2 * g + (d & 1);
      const uint32_t w0 = (((R << (l + 1)) + G) << (l - 4)) + 2 * k;
      lo |= child[w0];
      hi |= child[w0 + 1];
    }
    return fold_pairs(lo) | (fold_pairs(hi) << 16);
  }
  // l <= 4: the word holds 32/m parent rows of m bits (fewer for l = 1)
  const uint32_t m = 1u << l;
  const uint32_t rows = min(32u / m, (1u << (3 * l)) / m);
  const uint32_t cmask = (2 * m >= 32) ? 0xFFFFFFFFu : ((1u << (2 * m)) - 1u);
  uint32_t out = 0;
  for (uint32_t j = 0; j < rows; ++j) {
    const uint32_t row = ((32u * pw) >> l) + j;
    const uint32_t r = row >> l, g = row & (m - 1u);
    uint32_t acc = 0;
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const uint32_t R = 2 * r + (d >> 1), G = 2 * g + (d & 1);
      const uint32_t off = ((R << (l + 1)) + G) * (2 * m);
      acc |= (child[off >> 5] >> (off & 31u)) & cmask;
    }
    out |= fold_pairs(acc) << (j * m);
  }
  return out;
}

// Word pw of cube-order level L-1 from the build kernel's row-layout bitset
// (the child rows (2r+dr, 2g+dg) of each parent row, OR-ed and pair-folded as
// in reduce_cube_word).
template <int L>
__device__ __forceinline__ uint32_t level_below_from_smem(const uint32_t* s, uint32_t pw) {
  using S = Smem<L>;
  if constexpr (L == 6) {
    const uint32_t r = pw >> 5, g = pw & 31u;     // one level-5 row per word
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const uint32_t a = (2 * r + (d >> 1)) * S::ROWW + 2 * g + (d & 1);
      lo |= s[a];
      hi |= s[S::HALF + a];
    }
    return fold_pairs(lo) | (fold_pairs(hi) << 16);
  } else {
    constexpr uint32_t m = 1u << (L - 1);                       // parent row bits
    constexpr uint32_t rows = (32u / m) < m * m ? 32u / m : m * m;
    uint32_t out = 0;
#pragma unroll
    for (uint32_t j = 0; j < rows; ++j) {
      const uint32_t row = pw * (32u / m) + j;
      const uint32_t r = row / m, g = row % m;
      uint32_t acc = 0;
#pragma unroll
      for (int d = 0; d < 4; ++d) acc |= s[(2 * r + (d >> 1)) * S::ROWW + 2 * g + (d & 1)];
      out |= fold_pairs(acc & S::ROWMASK) << (j * m);
    }
    return out;
  }
}

// Shared-window address of the build kernel's dynamic shared memory: the
// kernel has no static shared variables and is launched without clusters,
// so its dynamic block starts right after the 1 KB reserved per CTA.  The
// kernel checks this once (trap otherwise); in exchange every lookup and
// atomic is [offset + immediate] -- a materialised base register costs an
// extra IADD per pixel.
constexpr uint32_t DYN_SMEM_BASE = 1024u;
__device__ __forceinline__ uint32_t lds_at(uint32_t off) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1+1024];" : "=r"(v) : "r"(off));
  return v;
}
__device__ __forceinline__ void reds_or_at(uint32_t off, uint32_t v) {
  asm volatile("red.shared.or.b32 [%0+1024], %1;" :: "r"(off), "r"(v) : "memory");
}
// ld.shared at [off] only where `skip` is 0; 0xFFFFFFFF (all present)
// elsewhere: a predicated-off lane adds no bank access to the wavefront
__device__ __forceinline__ uint32_t lds_at_unless(uint32_t off, uint32_t skip) {
  uint32_t v = 0xFFFFFFFFu;
  asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %2, 0;\n\t@p ld.shared.u32 %0, [%1+1024];\n\t}"
               : "+r"(v) : "r"(off), "r"(skip));
  return v;
}
// red.shared.or at [off] only in the lanes where `hit` is 0 (a predicated ATOMS)
__device__ __forceinline__ void reds_or_if(uint32_t off, uint32_t v, uint32_t hit) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %2, 0;\n\t@p red.shared.or.b32 [%0+1024], %1;\n\t}"
               :: "r"(off), "r"(v), "r"(hit) : "memory");
}

// bit 0 of v0 & v1 & v2 & v3 in two LOP3s (plain C++ lets ptxas share the
// v & 1 terms with the rare path and spend a third)
__device__ __forceinline__ bool all_hit4(const uint32_t (&v)[4]) {
  uint32_t t, u;
  asm("lop3.b32 %0, %1, %2, %3, 0x80;" : "=r"(t) : "r"(v[0]), "r"(v[1]), "r"(v[2]));
  asm("lop3.b32 %0, %1, %2, 1, 0x80;" : "=r"(u) : "r"(t), "r"(v[3]));
  return u != 0u;
}

// One 16-pixel unit, called by all 32 lanes of a warp (`valid` false for
// lanes past the segment).  Lookups go in groups of four; a group takes the
// atomic path only if some lane of the warp misses one of its pixels -- a
// warp-uniform branch, so the common path has no divergence (ncu r4-r6:
// per-pixel divergent branches cost ~5 instructions/pixel).  About 0.45 % of
// pixels miss at C3 (first occurrences of a colour within a CTA's range).
template <int L, bool SMEM_BITS, bool COUNTS, bool FULL>
__device__ __forceinline__ void build_unit(const uint32_t (&w)[12], uint32_t* bits, uint32_t* cnt,
                                           bool valid_) {
  // FULL: every lane of the warp holds a unit (the steady state); the tail
  // variant carries per-lane `valid`
  const bool valid = FULL || valid_;
  uint32_t px[16];
  unpack16<0, L>(w, px);
  char* base = reinterpret_cast<char*>(bits);
#pragma unroll
  for (int g = 0; g < 16; g += 4) {
    uint32_t addr[4], bsel[4], v[4];
    if constexpr (SMEM_BITS) {
      // byte offsets; the shared base rides in the LDS address ([R+UR])
      pair_positions_dyn<Smem<L>>(w, g / 2, 0u, addr[0], bsel[0], addr[1], bsel[1]);
      pair_positions_dyn<Smem<L>>(w, g / 2 + 1, 0u, addr[2], bsel[2], addr[3], bsel[3]);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t wd;
      if constexpr (SMEM_BITS) {
        wd = lds_at(addr[j]);
      } else {
        bit_position<L>(px[g + j], addr[j], bsel[j], 0u);
        wd = *reinterpret_cast<volatile uint32_t*>(base + addr[j]);
      }
      v[j] = __funnelshift_r(wd, wd, bsel[j]);
    }
    if constexpr (SMEM_BITS) {
      // Warp-uniform skip of the common all-hit group.  A slow group (about
      // a third of them at C3: first sightings of a leaf within the CTA's
      // segment are ~0.46 % of pixels, tools/sim_misses.py) issues four
      // predicated atomics, each landing only in the lanes that missed that
      // pixel: three instructions per pixel, no vote-reduce, no branches
      // per pixel (the REDUX + select version cost ~26 per slow group).
      const bool miss = valid && !all_hit4(v);
      if (__any_sync(0xFFFFFFFFu, miss)) {
#pragma unroll
        for (int j = 0; j < 4; ++j) reds_or_if(addr[j], Smem<L>::set_mask(bsel[j]), valid ? (v[j] & 1u) : 1u);
      }
    } else {
      const bool miss = valid && !(v[0] & v[1] & v[2] & v[3] & 1u);
      if (__any_sync(0xFFFFFFFFu, miss)) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (valid && !(v[j] & 1u)) atomicOr(reinterpret_cast<uint32_t*>(base + addr[j]), 1u << (bsel[j] & 31u));
      }
    }
  }
  if constexpr (COUNTS) {
    if (valid) {
#pragma unroll
      for (int j = 0; j < 16; ++j) count_code<L>(cnt, operand_to_cube<L>(px[j]));
    }
  }
}

// End of a tree segment: OR the CTA's non-zero bitset words into the tree's
// workspace cube `dst` and, for obg_build_model (levels_out), its cube-order
// levels L-1..1 into the tree's upper levels at dst + CW (OR of partial
// presence = presence of the union, so the segments of one tree combine
// with atomics).  Cube-order levels are a few instructions per word;
// path-order ones here cost 5.5x K1's flush (ncu r8), which is why those
// are made once, for the merged model.  Leaves the bitset zeroed.
// Levels L-2 .. 1 of a flushed segment by ONE warp, in registers: lane R
// holds the rows (R, G) of level P = L-1 (2^P bits each); a level is the
// OR of row pairs (G) and lane pairs (R, one shuffle) with adjacent bit pairs
// folded (B).  Replaces a chain of four block-wide passes with barriers
// (~1.5-2k cycles per level, clock64 r3) by ~100 instructions of one warp.
// Level-l words are OR-ed into `up` (cube-order level_offset layout).
template <int l, int P>
__device__ __forceinline__ void warp_levels_down(const uint32_t (&F)[2 << l], uint32_t* up, int lane) {
  constexpr int M = 1 << l;                        // rows along G (and bits per row) at level l
  uint32_t Fl[M];
#pragma unroll
  for (int g = 0; g < M; ++g) {
    uint32_t x = F[2 * g] | F[2 * g + 1];
    x |= __shfl_xor_sync(0xFFFFFFFFu, x, 1 << (P - 1 - l));
    Fl[g] = fold_pairs(x);                         // 2^l bits
  }
  // lanes with R_l = lane >> (P - l) and the low bits clear write row r
  if ((lane & ((1 << (P - l)) - 1)) == 0 && (lane >> (P - l)) < M) {
    const uint32_t r = uint32_t(lane >> (P - l));
    constexpr int RPW = 32 / M < M * M ? 32 / M : M * M;        // rows per word
    constexpr uint32_t off = uint32_t(level_offset(l));
#pragma unroll
    for (int g0 = 0; g0 < M; g0 += RPW) {
      const uint32_t row0 = r * M + uint32_t(g0);
      uint32_t w = 0;
#pragma unroll
      for (int j = 0; j < RPW && g0 + j < M; ++j) w |= Fl[g0 + j] << (j * M);
      const uint32_t bit0 = row0 * M;
      if (w) atomicOr(up + off + (bit0 >> 5), w << (bit0 & 31u));
    }
  }
  if constexpr (l > 1) warp_levels_down<l - 1, P>(Fl, up, lane);
}

// P = L-1 level words in the flush scratch `lv` (cube order) -> levels P-1..1.
template <int P>
__device__ __forceinline__ void warp_upper_levels(const uint32_t* lv, uint32_t* up, int lane) {
  constexpr int M = 1 << P;
  uint32_t F[M];
#pragma unroll
  for (int g = 0; g < M; ++g) {
    uint32_t x = 0;
    if (lane < M) {
      if constexpr (P == 5) x = lv[lane * 32 + g];                              // one row per word
      else x = (lv[(lane * M + g) >> 1] >> (16 * (g & 1))) & 0xFFFFu;           // P = 4: two rows per word
    }
    F[g] = x;
  }
  warp_levels_down<P - 1, P>(F, up, lane);
}

template <int L, int NT>
__device__ __forceinline__ void flush_segment(uint32_t* s_bits, uint32_t* dst, int levels_out, bool last) {
  __syncthreads();                                   // the segment's bitset is complete
  uint32_t* up = dst + cube_words(L);
  uint32_t* sc = s_bits + Smem<L>::SCRATCH;
  const bool levels = L >= 2 && levels_out;
  // phase A: level L-1 from the bitset (read only)
  if constexpr (L >= 2) {
    if (levels) {
      constexpr uint32_t NW = uint32_t(level_words(L - 1));
      constexpr uint32_t OFF = uint32_t(level_offset(L - 1));
      for (uint32_t pw = threadIdx.x; pw < NW; pw += NT) {
        const uint32_t v = level_below_from_smem<L>(s_bits, pw);
        sc[OFF + pw] = v;
        if (v) atomicOr(up + OFF + pw, v);
      }
      __syncthreads();
    }
  }
  // levels L-2..1 (L = 5, 6): warp 0 in registers, while the others start phase B
  constexpr bool WARP_LEVELS = L == 5 || L == 6;
  if constexpr (WARP_LEVELS) {
    if (levels && threadIdx.x < 32)
      warp_upper_levels<L - 1>(sc + level_offset(L - 1), up, int(threadIdx.x));
  }
  // phase B: OR the non-zero leaf words into the tree's cube and clear them
  // (data words only; the pads stay 0)
  for (uint32_t i = threadIdx.x; i < Smem<L>::data_words; i += NT) {
    const uint32_t p = Smem<L>::data_word(i);
    const uint32_t x = s_bits[p];
    if (x) {
      flush_smem_word<L>(dst, p, x);
      if (!last) s_bits[p] = 0u;
    }
  }
  if constexpr (L >= 3 && !WARP_LEVELS) {
    if (levels) {
      for (int l = L - 2; l >= 1; --l) {
        const uint32_t nw = uint32_t(level_words(l)), off = uint32_t(level_offset(l));
        const uint32_t* child = sc + level_offset(l + 1);
        for (uint32_t pw = threadIdx.x; pw < nw; pw += NT) {
          const uint32_t v = reduce_cube_word(child, l, pw);
          sc[off + pw] = v;
          if (v) atomicOr(up + off + pw, v);
        }
        __syncthreads();
      }
      return;
    }
  }
  __syncthreads();                                   // bitset clear before the next segment
}

#ifndef OBG_ALIGN_TREES
#define OBG_ALIGN_TREES 1
#endif
#ifndef OBG_BUILD_STAGES3
#define OBG_BUILD_STAGES3 1         // 0: two register buffers at every depth (A/B)
#endif
#ifndef OBG_BUILD_NOLOOKUP
#define OBG_BUILD_NOLOOKUP 0      // experiment: stream the frames without lookups (load-structure bound)
#endif
#ifndef OBG_BUILD_PF
#define OBG_BUILD_PF 0            // > 0: lane 0 bulk-prefetches the warp's chunk this many iterations ahead into L2
#endif
template <int L, bool SMEM_BITS, bool COUNTS>
__global__ void __launch_bounds__(BUILD_BLOCK, OBG_BUILD_MINB)
k_build_flat(const uint8_t* __restrict__ frames, int64_t units_per_frame, int64_t total_units,
             int group_size, int64_t units_per_cta, uint32_t* __restrict__ ws,
             uint32_t* __restrict__ out_pyr, int64_t n_trees, uint32_t* __restrict__ zero_cube,
             int64_t zero_words, uint32_t* __restrict__ counts, int levels_out) {
  // Smem<L>::alloc_words of dynamic shared memory (the bitset and the
  // per-lane dummy words); lookups address it as [offset + UR base]
  extern __shared__ __align__(1024) uint32_t s_bits[];
  if constexpr (SMEM_BITS) {
    if (static_cast<uint32_t>(__cvta_generic_to_shared(s_bits)) != DYN_SMEM_BASE) __trap();
  }
  if (gridDim.x <= PDL_EARLY_GRID) pdl_launch_dependents();   // SMs are free: the merge's CTAs may take them now
  constexpr int64_t CW = cube_words(L), WSW = ws_words(L);
  if (blockIdx.x == 0) {
    clear_shared_words(out_pyr, n_trees, L);
    for (int64_t i = threadIdx.x; i < zero_words; i += BUILD_BLOCK) zero_cube[i] = 0u;
  }
  const int64_t u_begin = int64_t(blockIdx.x) * units_per_cta;
  const int64_t u_end = min(total_units, u_begin + units_per_cta);
  if (u_begin >= u_end) return;
  if constexpr (SMEM_BITS) {
    for (uint32_t i = threadIdx.x; i < Smem<L>::compact; i += BUILD_BLOCK) s_bits[Smem<L>::compact_word(i)] = 0u;
    __syncthreads();
  }
  const int64_t units_per_tree = units_per_frame * group_size;
  int64_t u = u_begin;
  while (u < u_end) {
    const int64_t tree = u / units_per_tree;
    const int64_t seg_end = min(u_end, (tree + 1) * units_per_tree);
    uint32_t* bits;
    if constexpr (SMEM_BITS) bits = s_bits;
    else bits = ws + tree * WSW;
    uint32_t* cnt = COUNTS ? counts + tree * (int64_t(1) << (3 * L)) : nullptr;
    // Software-pipelined: the next unit's three 16-byte loads are in flight
    // while the current one is looked up (unrolled by two so the buffers
    // swap by renaming).  Trip counts are warp-uniform (lanes past the
    // segment carry valid=false) so build_unit can branch on warp votes.
    // 32-bit trip counts and a pointer bump per iteration: the 64-bit unit
    // indices cost ~1.2 instructions per pixel (ncu r18).
    const int lane = threadIdx.x & 31;
    const int64_t seg_len = seg_end - u;                               // < 2^31 (host checks units_per_cta)
    const int32_t rel0 = int32_t(threadIdx.x) - lane;                  // warp's first unit
    const int32_t n_it = seg_len > rel0 ? int32_t((seg_len - rel0 + BUILD_BLOCK - 1) / BUILD_BLOCK) : 0;
    const int32_t n_full = seg_len >= rel0 + 32 ? int32_t((seg_len - rel0 - 32) / BUILD_BLOCK) + 1 : 0;
    const int32_t n_lane = seg_len > rel0 + lane ? int32_t((seg_len - rel0 - lane + BUILD_BLOCK - 1) / BUILD_BLOCK) : 0;
    constexpr int64_t STEP = 48 * int64_t(BUILD_BLOCK);
    const uint8_t* fp = frames + 48 * (u + rel0 + lane);
#define OBG_BUILD_STEP(CUR, NXT)                                                              \
    {                                                                                          \
      if (OBG_BUILD_PF > 0 && lane == 0 && k + OBG_BUILD_PF < n_full)                          \
        prefetch_l2_bulk(fp + OBG_BUILD_PF * STEP, 48 * 32);                                   \
      if (k + STAGES - 1 < n_lane) load_unit_at(fp + (STAGES - 1) * STEP, NXT);                \
      if (OBG_BUILD_NOLOOKUP) {                                                                \
        _Pragma("unroll") for (int q_ = 0; q_ < 12; ++q_) sink ^= CUR[q_];                     \
      } else if (k < n_full) build_unit<L, SMEM_BITS, COUNTS, true>(CUR, bits, cnt, true);     \
      else build_unit<L, SMEM_BITS, COUNTS, false>(CUR, bits, cnt, k < n_lane);                \
      fp += STEP;                                                                              \
      ++k;                                                                                     \
    }
    // L = 6: three register buffers, two units in flight per thread while the
    // third is looked up.  ncu's source page puts 28 % of K1's stall samples on
    // the first use of a freshly loaded unit (profiles/r02_ncu_build_hot_lines.md);
    // the third buffer costs spills only outside the steady-state loop.  A/B
    // (profiles/ab_r02/r02_ab_stages3.txt): C3 model 80.5 -> 79.6 us, C4
    // constant L6 134.7 -> 131.7 us; L = 4 / 5 measured +-1 % and keep two.
    constexpr int STAGES = (L == 6 && OBG_BUILD_STAGES3) ? 3 : 2;
    uint32_t sink = 0;
    if constexpr (STAGES == 3) {
      uint32_t wa[12], wb[12], wc[12];
      if (0 < n_lane) load_unit_at(fp, wa);
      if (1 < n_lane) load_unit_at(fp + STEP, wb);
      for (int32_t k = 0; k < n_it;) {
        OBG_BUILD_STEP(wa, wc)
        if (k >= n_it) break;
        OBG_BUILD_STEP(wb, wa)
        if (k >= n_it) break;
        OBG_BUILD_STEP(wc, wb)
      }
    } else {
      uint32_t wa[12], wb[12];
      if (0 < n_lane) load_unit_at(fp, wa);
      for (int32_t k = 0; k < n_it;) {
        OBG_BUILD_STEP(wa, wb)
        if (k >= n_it) break;
        OBG_BUILD_STEP(wb, wa)
      }
    }
#undef OBG_BUILD_STEP
    if (OBG_BUILD_NOLOOKUP && sink == 0x9E3779B9u) ws[0] = sink;     // keep the loads (experiment only)
    if constexpr (SMEM_BITS) flush_segment<L, BUILD_BLOCK>(s_bits, ws + tree * WSW, levels_out, seg_end >= u_end);
    u = seg_end;
  }
}

// ---------------------------------------------------------------------------
// K1 with a region grid (R x C > 1, model.py:61-75, 93-109), L <= 6,
// W % 16 == 0: blockIdx.y = region row r (a band of rows); the CTA keeps one
// shared bitset per column region (C of them, BB bytes apart) and streams
// the band's units; at a tree (frame group) boundary it flushes bitset c into
// tree g * R * C + r * C + c.  A unit cut by a column boundary is handled per
// pixel by its lanes after the warp's vote-based pass (where they count as
// invalid), so warp collectives stay converged.
// ---------------------------------------------------------------------------
template <int L>
struct BandBits {
  static constexpr uint32_t ALLOC = (uint32_t(Smem<L>::alloc_words) + 31u) & ~31u;   // words per bitset
};

template <int L>
__device__ __forceinline__ void build_unit_band(const uint32_t (&w)[12], bool valid, uint32_t ob) {
#pragma unroll
  for (int g = 0; g < 16; g += 4) {
    uint32_t addr[4], bsel[4], v[4];
    pair_positions_dyn<Smem<L>>(w, g / 2, 0u, addr[0], bsel[0], addr[1], bsel[1]);
    pair_positions_dyn<Smem<L>>(w, g / 2 + 1, 0u, addr[2], bsel[2], addr[3], bsel[3]);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      addr[j] += ob;
      const uint32_t wd = lds_at(addr[j]);
      v[j] = __funnelshift_r(wd, wd, bsel[j]);
    }
    const bool miss = valid && !all_hit4(v);
    if (__any_sync(0xFFFFFFFFu, miss)) {
#pragma unroll
      for (int j = 0; j < 4; ++j) reds_or_if(addr[j], Smem<L>::set_mask(bsel[j]), valid ? (v[j] & 1u) : 1u);
    }
  }
}

// per pixel (a unit cut by a column boundary): pixel j at column x0 + j
template <int L>
__device__ __forceinline__ void build_unit_band_px(const uint32_t (&w)[12], int x0, const int* cb, int C) {
  uint32_t px[16];
  unpack16<0, L>(w, px);
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    int c = 0;
    while (c + 1 < C && x0 + j >= cb[c + 1]) ++c;
    uint32_t addr, bsel;
    bit_position<L, Smem<L>>(px[j], addr, bsel);
    addr += uint32_t(c) * (BandBits<L>::ALLOC * 4u);
    const uint32_t wd = lds_at(addr);
    reds_or_if(addr, Smem<L>::set_mask(bsel), __funnelshift_r(wd, wd, bsel) & 1u);
  }
}

template <int L>
__global__ void __launch_bounds__(BUILD_BLOCK, 1)
k_build_band(const uint8_t* __restrict__ frames, int n_frames_used, int H, int W, int R, int C, int group_size,
             int64_t per_cta, uint32_t* __restrict__ ws, uint32_t* __restrict__ out_pyr, int64_t n_trees,
             uint32_t* __restrict__ zero_cube, int64_t zero_words, int levels_out) {
  constexpr uint32_t ALLOC = BandBits<L>::ALLOC;
  constexpr int64_t WSW = ws_words(L);
  // dynamic smem only (the bitsets must start at DYN_SMEM_BASE): C bitsets,
  // then the C + 1 column boundaries
  extern __shared__ __align__(1024) uint32_t s_bits[];
  if (static_cast<uint32_t>(__cvta_generic_to_shared(s_bits)) != DYN_SMEM_BASE) __trap();
  int* s_cb = reinterpret_cast<int*>(s_bits + uint32_t(C) * ALLOC);
  if (blockIdx.x == 0 && blockIdx.y == 0) {
    clear_shared_words(out_pyr, n_trees, L);
    for (int64_t i = threadIdx.x; i < zero_words; i += BUILD_BLOCK) zero_cube[i] = 0u;
  }
  const int r = blockIdx.y;
  const int y0 = int((int64_t(r) * H + R - 1) / R), y1 = int((int64_t(r + 1) * H + R - 1) / R);
  const int W16 = W / 16;
  const int64_t band_units = int64_t(y1 - y0) * W16;
  const int64_t total = band_units * n_frames_used;
  const int64_t b_begin = int64_t(blockIdx.x) * per_cta;
  const int64_t b_end = min(total, b_begin + per_cta);
  if (b_begin >= b_end) return;
  if (threadIdx.x <= C) s_cb[threadIdx.x] = int((int64_t(threadIdx.x) * W + C - 1) / C);
  for (uint32_t c = 0; c < uint32_t(C); ++c)
    for (uint32_t i = threadIdx.x; i < Smem<L>::compact; i += BUILD_BLOCK) s_bits[c * ALLOC + Smem<L>::compact_word(i)] = 0u;
  __syncthreads();
  const int64_t upf = int64_t(H) * W16;
  const int64_t upt = band_units * group_size;                  // band units per tree
  const int lane = threadIdx.x & 31;
  const int32_t rel0 = int32_t(threadIdx.x) - lane;
  int64_t b = b_begin;
  while (b < b_end) {
    const int64_t grp = b / upt;
    const int64_t seg_end = min(b_end, (grp + 1) * upt);
    while (b < seg_end) {                                       // contiguous pieces: one frame each
      const int64_t f = b / band_units, k0 = b - f * band_units;
      const int64_t piece_end = min(seg_end, (f + 1) * band_units);
      const int64_t len = piece_end - b;
      const int64_t ubase = f * upf + int64_t(y0) * W16 + k0;
      const int32_t n_it = len > rel0 ? int32_t((len - rel0 + BUILD_BLOCK - 1) / BUILD_BLOCK) : 0;
      for (int32_t it = 0; it < n_it; ++it) {
        const int64_t rel = int64_t(it) * BUILD_BLOCK + rel0 + lane;
        const bool valid = rel < len;
        uint32_t w[12];
        if (valid) load_unit(frames, ubase + rel, w);
        else {
#pragma unroll
          for (int q = 0; q < 12; ++q) w[q] = 0u;
        }
        const int x0 = int((k0 + rel) % W16) * 16;
        int c = 0;
        while (c + 1 < C && x0 >= s_cb[c + 1]) ++c;
        const bool cut = x0 + 15 >= s_cb[c + 1];
        build_unit_band<L>(w, valid && !cut, uint32_t(c) * (ALLOC * 4u));
        if (valid && cut) build_unit_band_px<L>(w, x0, s_cb, C);
      }
      b = piece_end;
    }
    const bool last = seg_end >= b_end;
    for (int c = 0; c < C; ++c)
      flush_segment<L, BUILD_BLOCK>(s_bits + c * ALLOC, ws + (grp * R * C + int64_t(r) * C + c) * WSW, levels_out,
                                    last);
    if (last) break;
    __syncthreads();
  }
}

template <int L>
static int launch_build_band(const uint8_t* frames, int n_frames_used, int H, int W, int R, int C, int group_size,
                             uint32_t* ws, uint32_t* out_pyr, int64_t n_trees, uint32_t* zero_cube, int64_t zero_words,
                             cudaStream_t st, int levels_out) {
  const size_t smem = size_t(C) * BandBits<L>::ALLOC * 4 + 17 * 4;
  static DevCache attr_smem;
  if (int(smem) > attr_smem()) {
    CUDA_TRY(cudaFuncSetAttribute(k_build_band<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr_smem() = int(smem);
  }
  const int64_t band_units = (int64_t(H) / R + 1) * (W / 16);
  // one CTA per SM in total, R bands x per_band within ONE wave (rounding
  // up put 3 x 50 CTAs on 148 SMs: a second wave of two CTAs for the 3x4 grid)
  const int64_t per_band = std::max<int64_t>(1, int64_t(sm_count()) / R);
  int64_t per_cta = (band_units * n_frames_used + per_band - 1) / per_band;
  const int64_t min_per_cta = int64_t(BUILD_BLOCK) * 4;
  if (per_cta < min_per_cta) per_cta = min_per_cta;
  const int64_t gx = (band_units * n_frames_used + per_cta - 1) / per_cta;
  k_build_band<L><<<dim3(unsigned(gx), unsigned(R)), BUILD_BLOCK, smem, st>>>(
      frames, n_frames_used, H, W, R, C, group_size, per_cta, ws, out_pyr, n_trees, zero_cube, zero_words, levels_out);
  LAUNCH_CHECK("k_build_band");
  return OBG_OK;
}

// ---------------------------------------------------------------------------
// K1 for L = 5 (and 4) with a BYTE per leaf (32 / 4 KB table): a pixel's leaf
// is recorded with one plain byte store of 1 -- idempotent, so no lookup,
// no warp vote, no miss path and no atomics (the bit-per-leaf K1 spends
// ~8 instructions per pixel on lookup + test + vote, and its miss path on
// every first sighting).  Row layout: byte R' * RS + G' * GS + B', RS =
// 2^L * GS + 16 bytes (the 16-byte pad skews R' across banks; GS below).
// At a tree boundary the table is packed into the bit-per-leaf row layout
// (Smem<L>, right after the table) and flushed by flush_segment as before.
// ---------------------------------------------------------------------------
template <int L>
struct ByteTab {
  static constexpr int s = 8 - L;
  // bytes per G' row: L = 5 pads the 32-byte rows to 40 (10 words: G' rows
  // 16 apart share a bank instead of 4; the G' term becomes one IMAD by 5)
  static constexpr uint32_t GS = L == 5 ? 40u : (1u << L);
  static constexpr uint32_t RS = (1u << L) * GS + 16u;           // bytes per R' row
  static constexpr uint32_t BYTES = (1u << L) * RS;
  static constexpr uint32_t BITS_OFF = (BYTES + 1023u) & ~1023u;  // byte offset of the Smem<L> bitset
  static_assert(RS % (1u << s) == 0 && RS % 16 == 0 && GS % 8 == 0, "row strides");
};

// byte offsets of pixels 2K and 2K+1 of a unit in the table
template <int L, int K>
__device__ __forceinline__ void byte_pair(const uint32_t (&w)[12], uint32_t& a, uint32_t& b) {
  using T = ByteTab<L>;
  constexpr int s = T::s;
  constexpr uint32_t M = (1u << L) - 1u;
  constexpr int o = 6 * K, i = o >> 2, j = o & 3;
  constexpr uint32_t selR = uint32_t(j) | (uint32_t(j) << 4) | (uint32_t(j + 3) << 8) | (uint32_t(j + 3) << 12);
  constexpr uint32_t selG = uint32_t(j + 1) | (uint32_t(j + 2) << 4) | (uint32_t(j + 4) << 8) | (uint32_t(j + 5) << 12);
  const uint32_t yR = __byte_perm(w[i], w[i + 1], selR);           // [R_A, R_A, R_B, R_B]
  const uint32_t yG = __byte_perm(w[i], w[i + 1], selG);           // [G_A, B_A, G_B, B_B]
  const uint32_t P = yR & ((M << s) | (M << (s + 16)));            // R & ~(2^s-1) per half
  const uint32_t gq = yG & ((M << s) | (M << (s + 16)));           // G & ~(2^s-1): G' << s
  const uint32_t bq = (yG >> (8 + s)) & (M | (M << 16));           // B'
  uint32_t q;
  if constexpr (L == 5) q = gq * 5u + bq;                         // G' * 40 + B' (gq = G' << 3)
  else if constexpr (2 * L - 8 >= 0) q = (gq << (2 * L - 8)) | bq; // G' << L | B'
  else q = (gq >> (8 - 2 * L)) | bq;
  const uint32_t pair = P * (T::RS >> s) + q;
  b = __umulhi(pair, 1u << 16);
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(a) : "r"(b), "r"(0xFFFF0000u), "r"(pair));   // pair & 0xFFFF
}

__device__ __forceinline__ void sts_one(uint32_t off) {
  asm volatile("st.shared.u8 [%0+1024], %1;" :: "r"(off), "r"(1u) : "memory");
}

template <int L, bool FULL>
__device__ __forceinline__ void build_unit_bytes(const uint32_t (&w)[12], bool valid) {
  // lanes past the segment store nothing (a warp-uniform branch in the
  // steady state, FULL)
  if (!FULL && !valid) return;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    uint32_t a, b;
    switch (k) {
      case 0: byte_pair<L, 0>(w, a, b); break;
      case 1: byte_pair<L, 1>(w, a, b); break;
      case 2: byte_pair<L, 2>(w, a, b); break;
      case 3: byte_pair<L, 3>(w, a, b); break;
      case 4: byte_pair<L, 4>(w, a, b); break;
      case 5: byte_pair<L, 5>(w, a, b); break;
      case 6: byte_pair<L, 6>(w, a, b); break;
      default: byte_pair<L, 7>(w, a, b); break;
    }
    sts_one(a);
    sts_one(b);
  }
}

// 4 bytes of 0/1 -> 4 bits
__device__ __forceinline__ uint32_t pack4(uint32_t x) { return (x * 0x10204080u) >> 28; }

// Pack the byte table into the Smem<L> bit-per-leaf rows (and clear it).
template <int L>
__device__ __forceinline__ void pack_byte_table(uint32_t* s_tab, uint32_t* s_bits, bool clear) {
  using T = ByteTab<L>;
  using S = Smem<L>;
  constexpr uint32_t ROWS = 1u << (2 * L);                         // (R', G') rows of 2^L bytes
  for (uint32_t r = threadIdx.x; r < ROWS; r += BUILD_BLOCK) {
    const uint32_t R = r >> L, G = r & ((1u << L) - 1u);
    uint2* src = reinterpret_cast<uint2*>(reinterpret_cast<char*>(s_tab) + R * T::RS + G * T::GS);
    uint32_t bits = 0;
#pragma unroll
    for (int v = 0; v < (1 << L) / 8; ++v) {                      // 8-byte pieces (rows are 8-byte aligned)
      const uint2 q = src[v];
      bits |= (pack4(q.x) | (pack4(q.y) << 4)) << (8 * v);
      if (clear) src[v] = make_uint2(0u, 0u);
    }
    if constexpr (L == 5) s_bits[R * S::ROWW + G] = bits;
    else s_bits[R * S::ROWW + G] = bits * S::REP;                  // L = 4: 16-bit row replicated
  }
}

template <int L>
__global__ void __launch_bounds__(BUILD_BLOCK, OBG_BUILD_MINB)
k_build_bytes(const uint8_t* __restrict__ frames, int64_t units_per_frame, int64_t total_units,
              int group_size, int64_t units_per_cta, uint32_t* __restrict__ ws,
              uint32_t* __restrict__ out_pyr, int64_t n_trees, uint32_t* __restrict__ zero_cube,
              int64_t zero_words, int levels_out) {
  using T = ByteTab<L>;
  extern __shared__ __align__(1024) uint32_t s_tab[];
  if (static_cast<uint32_t>(__cvta_generic_to_shared(s_tab)) != DYN_SMEM_BASE) __trap();
  if (gridDim.x <= PDL_EARLY_GRID) pdl_launch_dependents();   // SMs are free: the merge's CTAs may take them now
  uint32_t* s_bits = s_tab + T::BITS_OFF / 4;
  constexpr int64_t WSW = ws_words(L);
  if (blockIdx.x == 0) {
    clear_shared_words(out_pyr, n_trees, L);
    for (int64_t i = threadIdx.x; i < zero_words; i += BUILD_BLOCK) zero_cube[i] = 0u;
  }
  const int64_t u_begin = int64_t(blockIdx.x) * units_per_cta;
  const int64_t u_end = min(total_units, u_begin + units_per_cta);
  if (u_begin >= u_end) return;
  for (uint32_t i = threadIdx.x; i < T::BYTES / 16; i += BUILD_BLOCK)
    reinterpret_cast<uint4*>(s_tab)[i] = make_uint4(0u, 0u, 0u, 0u);
  for (uint32_t i = threadIdx.x; i < Smem<L>::compact; i += BUILD_BLOCK) s_bits[Smem<L>::compact_word(i)] = 0u;
  __syncthreads();
  const int64_t units_per_tree = units_per_frame * group_size;
  int64_t u = u_begin;
  while (u < u_end) {
    const int64_t tree = u / units_per_tree;
    const int64_t seg_end = min(u_end, (tree + 1) * units_per_tree);
    const int lane = threadIdx.x & 31;
    const int64_t seg_len = seg_end - u;
    const int32_t rel0 = int32_t(threadIdx.x) - lane;
    const int32_t n_it = seg_len > rel0 ? int32_t((seg_len - rel0 + BUILD_BLOCK - 1) / BUILD_BLOCK) : 0;
    const int32_t n_full = seg_len >= rel0 + 32 ? int32_t((seg_len - rel0 - 32) / BUILD_BLOCK) + 1 : 0;
    const int32_t n_lane = seg_len > rel0 + lane ? int32_t((seg_len - rel0 - lane + BUILD_BLOCK - 1) / BUILD_BLOCK) : 0;
    constexpr int64_t STEP = 48 * int64_t(BUILD_BLOCK);
    const uint8_t* fp = frames + 48 * (u + rel0 + lane);
    uint32_t wa[12], wb[12];
    if (0 < n_lane) load_unit_at(fp, wa);
    for (int32_t k = 0; k < n_it;) {
      if (k + 1 < n_lane) load_unit_at(fp + STEP, wb);
      if (k < n_full) build_unit_bytes<L, true>(wa, true);
      else build_unit_bytes<L, false>(wa, k < n_lane);
      fp += STEP;
      if (++k >= n_it) break;
      if (k + 1 < n_lane) load_unit_at(fp + STEP, wa);
      if (k < n_full) build_unit_bytes<L, true>(wb, true);
      else build_unit_bytes<L, false>(wb, k < n_lane);
      fp += STEP;
      ++k;
    }
    const bool last = seg_end >= u_end;
    __syncthreads();                                  // the segment's table is complete
    pack_byte_table<L>(s_tab, s_bits, !last);
    flush_segment<L, BUILD_BLOCK>(s_bits, ws + tree * WSW, levels_out, last);
    u = seg_end;
  }
}

// ---------------------------------------------------------------------------
// K1 through a TMA ring (L <= 6).  Same segment streaming, lookups and flush
// as k_build_flat / k_build_bytes, but the frame bytes reach the SM by bulk
// async copies: one cp.async.bulk per CTA iteration (its 1024 units = 48 KB,
// contiguous in the frame batch) into a ring of RING_STAGES stages, each with
// an mbarrier; lanes read their 48-byte unit back with three conflict-free
// LDS.128.  Why (ncu r02 of k_build_flat<6>: L1/TEX 71 % busy, long-scoreboard
// the top stall, 60 % issue active):
//  * the register-pipelined kernel keeps one unit per thread in flight (49 KB
//    per SM, about what 6.4 TB/s x ~1.2 us needs with nothing to spare), the
//    ring RING_STAGES x 48 KB without a register;
//  * a 48-byte-strided LDG.128 touches 12 lines per warp instruction and the
//    three loads of a unit touch the same 12: 36 L1 tag wavefronts per 1536
//    bytes against 12 for the ring's LDS, and none for the bulk copy;
//  * the copies keep streaming across tree boundaries while the CTA flushes
//    its bitset, so the segment clear / flush / drain (~5 us at C3) overlaps.
// No producer warp: the warp that releases a stage LAST (a shared counter per
// stage) issues that stage's refill, RING_STAGES iterations ahead, so nobody
// waits for a slot.  tools/probes/ring_probe.cu: this ring streams 6.7 TB/s
// (the LDG pattern 6.4); a private 1.5 KB ring per warp only 2.6-3.6 TB/s
// (many small bulk copies in flight), which is why the ring is per CTA.
// ---------------------------------------------------------------------------
#ifndef OBG_RING_STAGES
#define OBG_RING_STAGES 3
#endif
#ifndef OBG_RING_RELAXED
#define OBG_RING_RELAXED 1        // stage release without a CTA fence (see ring_release)
#endif
#ifndef OBG_BUILD_RING
#define OBG_BUILD_RING 0          // 1: K1 through the TMA ring (A/B: slower, see above)
#endif
constexpr int RING_STAGES = OBG_RING_STAGES;

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "OBG_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@p bra OBG_DONE;\n\t"
      "bra OBG_WAIT;\n\t"
      "OBG_DONE:\n\t}"
      :: "r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void lds_unit(uint32_t addr, uint32_t (&w)[12]) {
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "r"(addr));
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4+16];" : "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]) : "r"(addr));
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4+32];" : "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]) : "r"(addr));
}
// release of a ring stage by one warp: returns how many warps released it before
__device__ __forceinline__ uint32_t ring_release(uint32_t cnt_addr) {
  uint32_t old;
#if OBG_RING_RELAXED
  asm volatile("atom.relaxed.cta.shared.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(cnt_addr) : "memory");
#else
  asm volatile("atom.acq_rel.cta.shared.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(cnt_addr) : "memory");
#endif
  return old;
}

// Shared-memory plan of k_build_ring: the table(s) of the lookup kernels at
// the dynamic base, then the ring stages, the mbarriers and the release counters.
template <int L, bool BYTES, int NT>
struct RingPlan {
  static constexpr uint32_t table_bytes() {
    if constexpr (BYTES) return ByteTab<L>::BITS_OFF + uint32_t(Smem<L>::alloc_words) * 4u;
    else return uint32_t(Smem<L>::alloc_words) * 4u;
  }
  static constexpr uint32_t STAGE = uint32_t(NT) * 48u;                 // one CTA iteration
  static constexpr uint32_t RING_OFF = (table_bytes() + 127u) & ~127u;
  static constexpr uint32_t BAR_OFF = RING_OFF + RING_STAGES * STAGE;
  static constexpr uint32_t CNT_OFF = BAR_OFF + RING_STAGES * 8u;
  static constexpr uint32_t CUR_OFF = (CNT_OFF + RING_STAGES * 4u + 15u) & ~15u;   // RingCursor per stage
  static constexpr uint32_t TOTAL = CUR_OFF + RING_STAGES * 24u;
  static_assert(TOTAL <= 227u * 1024u, "ring does not fit shared memory");
};

// The producer's position: the next CTA iteration (segment [u, end), k-th
// block of BUILD_BLOCK units) a stage will be refilled with.  One cursor per
// stage in shared memory, each stepping RING_STAGES iterations at a time, and
// touched only by the thread that refills that stage (refills of one stage are
// ordered by its mbarrier / release counter), so the streaming warps carry no
// producer state.
struct RingCursor {
  int64_t u, end;      // current segment (tree piece) of the CTA's range; u >= u_end: no more work
  int32_t k;           // iteration within the segment
  int32_t pad;
};
__device__ __forceinline__ void ring_advance(RingCursor& c, int64_t u_end, int64_t upt, int block) {
  if (c.u >= u_end) return;
  const int32_t n = int32_t((c.end - c.u + block - 1) / block);
  if (++c.k >= n) {
    c.u = c.end;
    c.end = min(u_end, c.u + upt);
    c.k = 0;
  }
}

template <int L, bool BYTES>
__global__ void __launch_bounds__(BUILD_BLOCK, 1)
k_build_ring(const uint8_t* __restrict__ frames, int64_t units_per_frame, int64_t total_units,
             int group_size, int64_t units_per_cta, uint32_t* __restrict__ ws,
             uint32_t* __restrict__ out_pyr, int64_t n_trees, uint32_t* __restrict__ zero_cube,
             int64_t zero_words, int levels_out) {
  using P = RingPlan<L, BYTES, BUILD_BLOCK>;
  constexpr uint32_t NW = BUILD_BLOCK / 32;
  extern __shared__ __align__(1024) uint32_t s_dyn[];
  if (static_cast<uint32_t>(__cvta_generic_to_shared(s_dyn)) != DYN_SMEM_BASE) __trap();
  if (gridDim.x <= PDL_EARLY_GRID) pdl_launch_dependents();   // SMs are free: the merge's CTAs may take them now
  uint32_t* s_bits = s_dyn;
  if constexpr (BYTES) s_bits = s_dyn + ByteTab<L>::BITS_OFF / 4;
  constexpr int64_t WSW = ws_words(L);
  const int lane = threadIdx.x & 31;
  const int32_t rel0 = int32_t(threadIdx.x) - lane;                    // warp's first unit of an iteration
  const int64_t u_begin = int64_t(blockIdx.x) * units_per_cta;
  const int64_t u_end = min(total_units, u_begin + units_per_cta);
  const int64_t upt = units_per_frame * group_size;                    // units per tree
  constexpr uint32_t ring0 = DYN_SMEM_BASE + P::RING_OFF;
  constexpr uint32_t bar0 = DYN_SMEM_BASE + P::BAR_OFF;
  constexpr uint32_t cnt0 = DYN_SMEM_BASE + P::CNT_OFF;
  RingCursor* s_cur = reinterpret_cast<RingCursor*>(reinterpret_cast<char*>(s_dyn) + P::CUR_OFF);

  // refill stage `slot` with its cursor's iteration and step the cursor (one thread)
  auto refill = [&](uint32_t slot) {
    RingCursor c = s_cur[slot];
    if (c.u >= u_end) return;
    const int64_t first = c.u + int64_t(c.k) * BUILD_BLOCK;
    const uint32_t bytes = uint32_t(min(int64_t(BUILD_BLOCK), c.end - first)) * 48u;
    mbar_expect_tx(bar0 + slot * 8u, bytes);
    bulk_g2s(ring0 + slot * P::STAGE, frames + 48 * first, bytes, bar0 + slot * 8u);
#pragma unroll
    for (int s = 0; s < RING_STAGES; ++s) ring_advance(c, u_end, upt, BUILD_BLOCK);
    s_cur[slot] = c;
  };

  if (u_begin < u_end && threadIdx.x == 0) {
    RingCursor c;
    c.u = u_begin;
    c.end = min(u_end, (u_begin / upt + 1) * upt);
    c.k = 0;
    c.pad = 0;
#pragma unroll
    for (int s = 0; s < RING_STAGES; ++s) {
      mbar_init(bar0 + s * 8u, 1u);
      s_dyn[P::CNT_OFF / 4 + s] = 0u;
      s_cur[s] = c;
      ring_advance(c, u_end, upt, BUILD_BLOCK);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#pragma unroll
    for (int s = 0; s < RING_STAGES; ++s) refill(uint32_t(s));         // in flight during the clears below
  }
  if (blockIdx.x == 0) {
    clear_shared_words(out_pyr, n_trees, L);
    for (int64_t i = threadIdx.x; i < zero_words; i += BUILD_BLOCK) zero_cube[i] = 0u;
  }
  if (u_begin >= u_end) return;
  if constexpr (BYTES) {
    for (uint32_t i = threadIdx.x; i < ByteTab<L>::BYTES / 16; i += BUILD_BLOCK)
      reinterpret_cast<uint4*>(s_dyn)[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  for (uint32_t i = threadIdx.x; i < Smem<L>::compact; i += BUILD_BLOCK) s_bits[Smem<L>::compact_word(i)] = 0u;
  __syncthreads();                                                     // tables clear, barriers initialised

  uint32_t c_slot = 0, c_phase = 0;
  const uint32_t unit_off = ring0 + uint32_t(threadIdx.x) * 48u;
  // take this warp's unit of the next CTA iteration out of the ring, release
  // the stage and (last warp out) refill it
  auto fetch = [&](uint32_t (&w)[12], bool any) {
    mbar_wait(bar0 + c_slot * 8u, c_phase);
    if (any) lds_unit(unit_off + c_slot * P::STAGE, w);
    __syncwarp();                                                      // every lane holds its unit
    if (lane == 0 && ring_release(cnt0 + c_slot * 4u) == NW - 1u) {
      s_dyn[P::CNT_OFF / 4 + c_slot] = 0u;
      refill(c_slot);
    }
    if (++c_slot == RING_STAGES) { c_slot = 0; c_phase ^= 1u; }
  };
  int64_t u = u_begin;
  int64_t seg_end = min(u_end, (u_begin / upt + 1) * upt);
  while (u < u_end) {
    const int64_t tree = u / upt;
    const int32_t seg_len = int32_t(seg_end - u);                      // < 2^31 (host checks units_per_cta)
    const int32_t n_it = (seg_len + BUILD_BLOCK - 1) / BUILD_BLOCK;
    int32_t left = seg_len - rel0;                                     // units from this warp's first to the segment end
    // the next unit comes out of the ring while the current one is looked up
    // (two register buffers swapped by unrolling, as in k_build_flat)
#define OBG_RING_STEP(CUR, NXT)                                                               \
    {                                                                                          \
      if (k + 1 < n_it) fetch(NXT, left > BUILD_BLOCK);                                        \
      if (left >= 32) {                                                                        \
        if constexpr (BYTES) build_unit_bytes<L, true>(CUR, true);                             \
        else build_unit<L, true, false, true>(CUR, s_bits, nullptr, true);                     \
      } else if (left > 0) {                                                                   \
        if constexpr (BYTES) build_unit_bytes<L, false>(CUR, lane < left);                     \
        else build_unit<L, true, false, false>(CUR, s_bits, nullptr, lane < left);             \
      }                                                                                        \
      left -= BUILD_BLOCK;                                                                     \
      ++k;                                                                                     \
    }
    uint32_t wa[12], wb[12];
    fetch(wa, left > 0);
    for (int32_t k = 0; k < n_it;) {
      OBG_RING_STEP(wa, wb)
      if (k >= n_it) break;
      OBG_RING_STEP(wb, wa)
    }
#undef OBG_RING_STEP
    const bool last = seg_end >= u_end;
    if constexpr (BYTES) {
      __syncthreads();                                                 // the segment's table is complete
      pack_byte_table<L>(s_dyn, s_bits, !last);
    }
    flush_segment<L, BUILD_BLOCK>(s_bits, ws + tree * WSW, levels_out, last);
    u = seg_end;
    seg_end = min(u_end, u + upt);
  }
}

// ---------------------------------------------------------------------------
// K1, L = 7: the 2^21-bit leaf set (256 KB) does not fit shared memory, so
// the CTA streams its range twice, once per half of the cube (R' top bit h),
// with that half (128 KB, skewed rows: R' & 63 x 128 G' x 4 B' words + pad)
// in shared memory; pixels of the other half count as hits.  Two frame reads
// instead of a global check-before-set per pixel: on uniform-random frames
// (~2 M distinct leaves per frame) the global bitset path made every lookup
// an L2 round trip and every first sight of a leaf a global atomic (r1:
// 0.07 of HBM).  1024 threads, one CTA per SM.
// ---------------------------------------------------------------------------
constexpr int L7H_BLOCK = 1024;
constexpr uint32_t L7H_ROWW = 512 + 5;                 // words per R' row (128 G' x 4) + pad
constexpr uint32_t L7H_WORDS = 64 * L7H_ROWW;          // one half of the cube
constexpr uint32_t L7H_ALLOC = L7H_WORDS + 32;         // + per-lane dummy words


// Returns nonzero if some pixel of the unit lies in the other half (so the
// CTA needs its second pass).
// Half-cube word offsets of pixels 2K and 2K+1, two at a time (as
// pair_positions): word offsets R6 * ROWW + G' * 4 + B' >> 5 are < 64 K, so
// both ride in the 16-bit halves of one register; byte addresses come out of
// the split.  mis_* bit 0 = the pixel lies in the other half (a "hit").
template <int K>
__device__ __forceinline__ void l7h_pair(const uint32_t (&w)[12], uint32_t hmask, uint32_t& addr_a, uint32_t& bsel_a,
                                         uint32_t& mis_a, uint32_t& addr_b, uint32_t& bsel_b, uint32_t& mis_b) {
  constexpr int o = 6 * K, a = o >> 2, b = o & 3;
  constexpr uint32_t selR = uint32_t(b) | (uint32_t(b) << 4) | (uint32_t(b + 3) << 8) | (uint32_t(b + 3) << 12);
  constexpr uint32_t selG = uint32_t(b + 1) | (uint32_t(b + 2) << 4) | (uint32_t(b + 4) << 8) | (uint32_t(b + 5) << 12);
  const uint32_t yR = __byte_perm(w[a], w[a + 1], selR);                 // [R_A, R_A, R_B, R_B]
  const uint32_t yG = __byte_perm(w[a], w[a + 1], selG);                 // [G_A, B_A, G_B, B_B]
  const uint32_t P = __umulhi(yR, 1u << 31) & 0x003F003Fu;               // (R >> 1) & 63 per half
  const uint32_t bq = __umulhi(yG, 1u << 18) & 0x00030003u;              // B >> 6 per half
  const uint32_t q = (yG & 0x00FE00FEu) * 2u + bq;                       // G' * 4 + B' >> 5
  const uint32_t pair = P * L7H_ROWW + q;                                // word offsets
  addr_b = __umulhi(pair, 1u << 18) & ~3u;                               // (pair >> 16) * 4
  addr_a = (pair << 2) & 0x3FFFCu;                                       // (pair & 0xFFFF) * 4
  bsel_a = __umulhi(yG, 1u << 23);                                       // yG >> 9: B_A' low bits
  bsel_b = __umulhi(yG, 1u << 7);                                        // yG >> 25
  const uint32_t hx = yR ^ hmask;                                        // R top bit vs the pass's half
  mis_a = hx >> 7;
  mis_b = hx >> 23;
}

template <int K>
__device__ __forceinline__ void l7h_pair_dyn(const uint32_t (&w)[12], int k, uint32_t hmask, uint32_t& aa,
                                             uint32_t& ba, uint32_t& ma, uint32_t& ab, uint32_t& bb, uint32_t& mb) {
  switch (k) {
    case 0: l7h_pair<0>(w, hmask, aa, ba, ma, ab, bb, mb); break;
    case 1: l7h_pair<1>(w, hmask, aa, ba, ma, ab, bb, mb); break;
    case 2: l7h_pair<2>(w, hmask, aa, ba, ma, ab, bb, mb); break;
    case 3: l7h_pair<3>(w, hmask, aa, ba, ma, ab, bb, mb); break;
    case 4: l7h_pair<4>(w, hmask, aa, ba, ma, ab, bb, mb); break;
    case 5: l7h_pair<5>(w, hmask, aa, ba, ma, ab, bb, mb); break;
    case 6: l7h_pair<6>(w, hmask, aa, ba, ma, ab, bb, mb); break;
    default: l7h_pair<7>(w, hmask, aa, ba, ma, ab, bb, mb); break;
  }
}

__device__ __forceinline__ uint32_t build_unit_l7h(const uint32_t (&w)[12], uint32_t hpass, bool valid) {
  uint32_t other = 0;
  const uint32_t hmask = hpass ? 0xFFFFFFFFu : 0u;
#pragma unroll
  for (int g = 0; g < 16; g += 4) {
    uint32_t addr[4], bsel[4], v[4], mis[4];
    l7h_pair_dyn<0>(w, g / 2, hmask, addr[0], bsel[0], mis[0], addr[1], bsel[1], mis[1]);
    l7h_pair_dyn<0>(w, g / 2 + 1, hmask, addr[2], bsel[2], mis[2], addr[3], bsel[3], mis[3]);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      // pixels of the other half are hits and do not touch shared memory
      // (uniform-random frames: half the lookups, fewer bank conflicts)
      const uint32_t wd = lds_at_unless(addr[j], mis[j] & 1u);
      v[j] = __funnelshift_r(wd, wd, bsel[j]) | mis[j];
    }
    const bool miss = valid && !(v[0] & v[1] & v[2] & v[3] & 1u);
    if (__any_sync(0xFFFFFFFFu, miss)) {
#pragma unroll
      for (int j = 0; j < 4; ++j) reds_or_if(addr[j], 1u << (bsel[j] & 31u), valid ? (v[j] & 1u) : 1u);
    }
  }
  // R bytes of the 16 pixels sit at bytes 0, 3, 6, 9 of each 12-byte group:
  // top bits 0x80000080 / 0x00800000 / 0x00008000 of words 3q, 3q+1, 3q+2
  const uint32_t x0 = hpass ? 0xFFFFFFFFu : 0u;
  const uint32_t o0 = (w[0] ^ x0) | (w[3] ^ x0) | (w[6] ^ x0) | (w[9] ^ x0);
  const uint32_t o1 = (w[1] ^ x0) | (w[4] ^ x0) | (w[7] ^ x0) | (w[10] ^ x0);
  const uint32_t o2 = (w[2] ^ x0) | (w[5] ^ x0) | (w[8] ^ x0) | (w[11] ^ x0);
  other = (o0 & 0x80000080u) | (o1 & 0x00800000u) | (o2 & 0x00008000u);
  return valid ? other : 0u;
}

__global__ void __launch_bounds__(L7H_BLOCK, 1)
k_build_l7h(const uint8_t* __restrict__ frames, int64_t units_per_frame, int64_t total_units, int group_size,
            int64_t units_per_cta, uint32_t* __restrict__ ws, uint32_t* __restrict__ out_pyr, int64_t n_trees,
            uint32_t* __restrict__ zero_cube, int64_t zero_words) {
  extern __shared__ __align__(1024) uint32_t s_bits[];
  if (static_cast<uint32_t>(__cvta_generic_to_shared(s_bits)) != DYN_SMEM_BASE) __trap();
  constexpr int64_t WSW = ws_words(7);
  if (blockIdx.x == 0) {
    clear_shared_words(out_pyr, n_trees, 7);
    for (int64_t i = threadIdx.x; i < zero_words; i += L7H_BLOCK) zero_cube[i] = 0u;
  }
  const int64_t u_begin = int64_t(blockIdx.x) * units_per_cta;
  const int64_t u_end = min(total_units, u_begin + units_per_cta);
  if (u_begin >= u_end) return;
  for (uint32_t i = threadIdx.x; i < L7H_WORDS; i += L7H_BLOCK) s_bits[i] = 0u;
  __syncthreads();
  const int64_t upt = units_per_frame * group_size;
  const int lane = threadIdx.x & 31;
  // First pass: the half of the range's first pixel (R' top bit = R >> 7);
  // the second pass only if the first one met a pixel of the other half
  // (a constant or dark scene needs one read of its frames, not two).
  const uint32_t h_first = uint32_t(__ldg(frames + 48 * u_begin)) >> 7;
  uint32_t need_other = 0;
  for (uint32_t pass = 0; pass < 2; ++pass) {
    if (pass == 1 && !__syncthreads_or(int(need_other))) break;
    const uint32_t h = pass == 0 ? h_first : 1u - h_first;
    int64_t u = u_begin;
    while (u < u_end) {
      const int64_t tree = u / upt;
      const int64_t seg_end = min(u_end, (tree + 1) * upt);
      // 32-bit trip counts and a pointer bump per iteration (as k_build_flat)
      const int64_t seg_len = seg_end - u;
      const int32_t rel0 = int32_t(threadIdx.x) - lane;
      const int32_t n_it = seg_len > rel0 ? int32_t((seg_len - rel0 + L7H_BLOCK - 1) / L7H_BLOCK) : 0;
      const int32_t n_lane =
          seg_len > rel0 + lane ? int32_t((seg_len - rel0 - lane + L7H_BLOCK - 1) / L7H_BLOCK) : 0;
      constexpr int64_t STEP = 48 * int64_t(L7H_BLOCK);
      const uint8_t* fp = frames + 48 * (u + rel0 + lane);
      uint32_t wa[12], wb[12];
      if (0 < n_lane) load_unit_at(fp, wa);
      for (int32_t k = 0; k < n_it;) {
        if (k + 1 < n_lane) load_unit_at(fp + STEP, wb);
        need_other |= build_unit_l7h(wa, h, k < n_lane);
        fp += STEP;
        if (++k >= n_it) break;
        if (k + 1 < n_lane) load_unit_at(fp + STEP, wa);
        need_other |= build_unit_l7h(wb, h, k < n_lane);
        fp += STEP;
        ++k;
      }
      // flush this half of the tree's leaf cube, leave the half-cube zeroed
      __syncthreads();
      uint32_t* dst = ws + tree * WSW;
      for (uint32_t p = threadIdx.x; p < L7H_WORDS; p += L7H_BLOCK) {
        const uint32_t x = s_bits[p];
        if (x) {
          const uint32_t r6 = p / L7H_ROWW, c = p - r6 * L7H_ROWW;          // c < 512: pads stay 0
          atomicOr(dst + (((64u * h + r6) << 9) | c), x);
          s_bits[p] = 0u;
        }
      }
      __syncthreads();
      u = seg_end;
    }
  }
}

// ---------------------------------------------------------------------------
// L = 7 build, ONE pass: 7/8 of the tree's 256 KB leaf set -- 112 of the 128
// R' slabs (512 words each, word index XOR-swizzled by the slab's low bits so
// R' varies the bank) -- in shared memory (224 KB; fewer slabs, leaving L1
// to the frame loads, measured slower: 96 / 80 / 64 slabs +13 / +40 / +63 %
// on uniform frames); the other 16 slabs, a
// window chosen per CTA opposite the R' of its range's first pixel (so a
// single-colour scene never lands there), straight in the tree's workspace
// cube in global memory (checked through L1, set with atomics: a stale L1
// copy only costs a redundant atomic).  Shared slab s holds R' = (s + 16 +
// g0) & 127.  Word offsets of a pixel pair ride in the two 16-bit halves of
// one register (slab << 9 | swizzled in-slab word < 65536) as in K1.
// k_build_l7h instead streams its range once per cube half (two frame reads).
// 1024 threads, one CTA per SM, dynamic smem at the fixed 1 KB window.
// ---------------------------------------------------------------------------
constexpr int L7C_BLOCK = 1024;
#ifndef OBG_L7B_SLABS
#define OBG_L7B_SLABS 112        // R' slabs (of 128) in shared memory; the rest is left to L1 for the frame loads
#endif
constexpr uint32_t L7C_N = OBG_L7B_SLABS;
constexpr uint32_t L7C_W = 128u - L7C_N;                 // global window
constexpr uint32_t L7C_WORDS = L7C_N * 512u;

// pixels 2K, 2K+1: byte addresses in shared memory (valid where !far),
// rotate amounts of the leaf bit, far flags (bit 0) and packed R' / in-row
// words for the global path.  k7 = ((L7C_N - g0) & 127) * 0x00010001.
template <int K>
__device__ __forceinline__ void l7c_pair(const uint32_t (&w)[12], uint32_t k7, uint32_t& addr_a, uint32_t& addr_b,
                                         uint32_t& bsel_a, uint32_t& bsel_b, uint32_t& far_a, uint32_t& far_b,
                                         uint32_t& rq, uint32_t& q) {
  constexpr int o = 6 * K, a = o >> 2, b = o & 3;
  constexpr uint32_t selR = uint32_t(b) | (uint32_t(b) << 4) | (uint32_t(b + 3) << 8) | (uint32_t(b + 3) << 12);
  constexpr uint32_t selG = uint32_t(b + 1) | (uint32_t(b + 2) << 4) | (uint32_t(b + 4) << 8) | (uint32_t(b + 5) << 12);
  const uint32_t yR = __byte_perm(w[a], w[a + 1], selR);                 // [R_A, R_A, R_B, R_B]
  const uint32_t yG = __byte_perm(w[a], w[a + 1], selG);                 // [G_A, B_A, G_B, B_B]
  rq = __umulhi(yR, 1u << 31) & 0x007F007Fu;                             // R' per half
  const uint32_t P = (rq + k7) & 0x007F007Fu;                            // shared slab (+ 112 .. 127: far)
  const uint32_t bq = __umulhi(yG, 1u << 18) & 0x00030003u;              // B >> 6 per half
  q = (yG & 0x00FE00FEu) * 2u + bq;                                      // G' * 4 + B' >> 5 per half
  const uint32_t pair = (P << 9) | (q ^ (P & 0x001F001Fu));              // swizzled word offsets
  addr_a = (pair << 2) & 0x3FFFCu;
  addr_b = __umulhi(pair, 1u << 18) & ~3u;
  bsel_a = __umulhi(yG, 1u << 23);
  bsel_b = __umulhi(yG, 1u << 7);
  far_a = (P & 0x7Fu) >= L7C_N;
  far_b = (P >> 16) >= L7C_N;
}

// `blind` (warp-uniform): set every pixel's bit without looking it up first.
// Check-before-set pays when most pixels hit; on frames whose pixels mostly
// miss (uniform-random 4K frames at L = 7: 2 M leaves, ~60 % first sightings
// per CTA segment) every group takes both the lookups and the atomics, 44
// instructions per pixel; the blind form is ~13.  The kernel switches per warp
// on the miss count of the last checked unit (`nmiss`, see k_build_l7c).
template <int K>
__device__ __forceinline__ void build_pairs_l7c(const uint32_t (&w)[12], bool valid, uint32_t k7,
                                                uint32_t* __restrict__ gcube, bool blind, uint32_t& nmiss) {
  uint32_t ad[4], bs[4], fr[4], v[4], go[4];
  {
    uint32_t rq0, q0, rq1, q1;
    l7c_pair<K>(w, k7, ad[0], ad[1], bs[0], bs[1], fr[0], fr[1], rq0, q0);
    l7c_pair<K + 1>(w, k7, ad[2], ad[3], bs[2], bs[3], fr[2], fr[3], rq1, q1);
    go[0] = ((rq0 & 0x7Fu) << 11) | ((q0 & 0xFFFFu) << 2);              // canonical cube byte offsets
    go[1] = ((rq0 >> 16) << 11) | ((q0 >> 16) << 2);
    go[2] = ((rq1 & 0x7Fu) << 11) | ((q1 & 0xFFFFu) << 2);
    go[3] = ((rq1 >> 16) << 11) | ((q1 >> 16) << 2);
  }
  if (blind) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (valid) {
        const uint32_t bit = 1u << (bs[j] & 31u);
        if (!fr[j]) reds_or_at(ad[j], bit);
        else atomicOr(reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(gcube) + go[j]), bit);
      }
    }
    return;
  }
  if (!__any_sync(0xFFFFFFFFu, (fr[0] | fr[1] | fr[2] | fr[3]) != 0u)) {
    // no pixel of the warp's 4-pixel group in the global window (the common
    // case away from the window, e.g. a single-colour scene): shared only
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t wd = lds_at(ad[j]);
      v[j] = __funnelshift_r(wd, wd, bs[j]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t wd;
      if (!fr[j]) wd = lds_at(ad[j]);
      else wd = __ldca(reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(gcube) + go[j]));
      v[j] = __funnelshift_r(wd, wd, bs[j]);
    }
  }
  const bool miss = valid && !(v[0] & v[1] & v[2] & v[3] & 1u);
  if (__any_sync(0xFFFFFFFFu, miss)) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (valid && !(v[j] & 1u)) {
        const uint32_t bit = 1u << (bs[j] & 31u);
        ++nmiss;
        if (!fr[j]) reds_or_at(ad[j], bit);
        else atomicOr(reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(gcube) + go[j]), bit);
      }
    }
  }
}

// Per-warp mode of the one-pass L7 build: a checked unit counts its missed
// pixels; above L7C_BLIND_MISSES of the warp's 512 the next L7C_BLIND_RUN units
// go blind, then one checked unit measures again.
#ifndef OBG_L7_BLIND
#define OBG_L7_BLIND 1
#endif
constexpr uint32_t L7C_BLIND_MISSES = 160;       // ~31 % of a warp-unit's pixels
#ifndef OBG_L7_BLIND_RUN
#define OBG_L7_BLIND_RUN 16
#endif
#ifndef OBG_L7_BLIND_THR
#define OBG_L7_BLIND_THR 8
#endif
constexpr int L7C_BLIND_RUN = OBG_L7_BLIND_RUN;
struct L7Mode {
  int blind_left = 0;
};
__device__ __forceinline__ void build_unit_l7c(const uint32_t (&w)[12], bool valid, uint32_t k7,
                                               uint32_t* __restrict__ gcube, L7Mode& mode) {
  uint32_t nmiss = 0;
  if (OBG_L7_BLIND && mode.blind_left > 0) {                     // warp-uniform
    build_pairs_l7c<0>(w, valid, k7, gcube, true, nmiss);
    build_pairs_l7c<2>(w, valid, k7, gcube, true, nmiss);
    build_pairs_l7c<4>(w, valid, k7, gcube, true, nmiss);
    build_pairs_l7c<6>(w, valid, k7, gcube, true, nmiss);
    --mode.blind_left;
    return;
  }
  build_pairs_l7c<0>(w, valid, k7, gcube, false, nmiss);
  build_pairs_l7c<2>(w, valid, k7, gcube, false, nmiss);
  build_pairs_l7c<4>(w, valid, k7, gcube, false, nmiss);
  build_pairs_l7c<6>(w, valid, k7, gcube, false, nmiss);
  // a lane with 5+ missed pixels of its 16 stands for a warp-unit above ~30 %
  // (misses spread evenly over the lanes of uniform-random frames; a natural
  // scene's few first sightings stay below)
  if (OBG_L7_BLIND && __any_sync(0xFFFFFFFFu, nmiss >= uint32_t(OBG_L7_BLIND_THR))) mode.blind_left = L7C_BLIND_RUN;
}

__global__ void __launch_bounds__(L7C_BLOCK, 1)
k_build_l7c(const uint8_t* __restrict__ frames, int64_t units_per_frame, int64_t total_units, int group_size,
            int64_t units_per_cta, uint32_t* __restrict__ ws, uint32_t* __restrict__ out_pyr, int64_t n_trees,
            uint32_t* __restrict__ zero_cube, int64_t zero_words) {
  extern __shared__ __align__(1024) uint32_t s_bits[];
  if (static_cast<uint32_t>(__cvta_generic_to_shared(s_bits)) != DYN_SMEM_BASE) __trap();
  constexpr int64_t WSW = ws_words(7);
  if (blockIdx.x == 0) {
    clear_shared_words(out_pyr, n_trees, 7);
    for (int64_t i = threadIdx.x; i < zero_words; i += L7C_BLOCK) zero_cube[i] = 0u;
  }
  const int64_t u_begin = int64_t(blockIdx.x) * units_per_cta;
  const int64_t u_end = min(total_units, u_begin + units_per_cta);
  if (u_begin >= u_end) return;
  for (uint32_t i = threadIdx.x; i < L7C_WORDS; i += L7C_BLOCK) s_bits[i] = 0u;
  __syncthreads();
  // the global window: L7C_W R' slabs opposite the R' of the range's first pixel
  const uint32_t g0 = ((uint32_t(__ldg(frames + 48 * u_begin)) >> 1) + 64u - L7C_W / 2u) & 127u;
  const uint32_t k7 = ((L7C_N - g0) & 127u) * 0x00010001u;
  const int64_t upt = units_per_frame * group_size;
  const int lane = threadIdx.x & 31;
  int64_t u = u_begin;
  while (u < u_end) {
    const int64_t tree = u / upt;
    const int64_t seg_end = min(u_end, (tree + 1) * upt);
    uint32_t* dst = ws + tree * WSW;
    const int64_t seg_len = seg_end - u;
    const int32_t rel0 = int32_t(threadIdx.x) - lane;
    const int32_t n_it = seg_len > rel0 ? int32_t((seg_len - rel0 + L7C_BLOCK - 1) / L7C_BLOCK) : 0;
    const int32_t n_lane = seg_len > rel0 + lane ? int32_t((seg_len - rel0 - lane + L7C_BLOCK - 1) / L7C_BLOCK) : 0;
    constexpr int64_t STEP = 48 * int64_t(L7C_BLOCK);
    const uint8_t* fp = frames + 48 * (u + rel0 + lane);
    uint32_t wa[12], wb[12];
    L7Mode mode;                                                  // a fresh segment starts checked
    if (0 < n_lane) load_unit_at(fp, wa);
    for (int32_t k = 0; k < n_it;) {
      if (k + 1 < n_lane) load_unit_at(fp + STEP, wb);
      build_unit_l7c(wa, k < n_lane, k7, dst, mode);
      fp += STEP;
      if (++k >= n_it) break;
      if (k + 1 < n_lane) load_unit_at(fp + STEP, wa);
      build_unit_l7c(wb, k < n_lane, k7, dst, mode);
      fp += STEP;
      ++k;
    }
    // flush the shared slabs into the tree's leaf cube, leave them zeroed
    __syncthreads();
    for (uint32_t p = threadIdx.x; p < L7C_WORDS; p += L7C_BLOCK) {
      const uint32_t x = s_bits[p];
      if (x) {
        const uint32_t sl = p >> 9, c = (p & 511u) ^ (sl & 31u);
        const uint32_t r = (sl + L7C_W + g0) & 127u;              // the slab's R'
        atomicOr(dst + ((r << 9) | c), x);
        s_bits[p] = 0u;
      }
    }
    __syncthreads();
    u = seg_end;
  }
}

// Generic path: any grid, any frame size / alignment.  One thread per pixel,
// region via region_of (model.py:61-66), bits in the workspace (global).
template <bool COUNTS>
__global__ void __launch_bounds__(256)
k_build_generic(const uint8_t* __restrict__ frames, int64_t n_pixels_used, int H, int W, int L,
                int R, int C, int group_size, uint32_t* __restrict__ ws, uint32_t* __restrict__ out_pyr,
                int64_t n_trees, uint32_t* __restrict__ zero_cube, int64_t zero_words,
                uint32_t* __restrict__ counts) {
  if (blockIdx.x == 0) {
    clear_shared_words(out_pyr, n_trees, L);
    for (int64_t i = threadIdx.x; i < zero_words; i += blockDim.x) zero_cube[i] = 0u;
  }
  const int64_t P = int64_t(H) * W;
  const int64_t CW = cube_words(L);
  const int s = 8 - L;
  const uint32_t m = (1u << L) - 1u;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n_pixels_used;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t f = i / P, p = i - f * P;
    const int y = int(p / W), x = int(p - int64_t(y) * W);
    const int row = min(R - 1, int(int64_t(y) * R / H));
    const int col = min(C - 1, int(int64_t(x) * C / W));
    const int64_t tree = (f / group_size) * (int64_t(R) * C) + int64_t(row) * C + col;
    const uint8_t* px = frames + 3 * i;
    const uint32_t idx = ((uint32_t(px[0]) >> s) << (2 * L)) | ((uint32_t(px[1]) >> s) << L) |
                         ((uint32_t(px[2]) >> s) & m);
    uint32_t* wp = ws + tree * ws_words(L) + (idx >> 5);
    if (!((*reinterpret_cast<volatile uint32_t*>(wp) >> (idx & 31u)) & 1u)) atomicOr(wp, 1u << (idx & 31u));
    if (COUNTS) {
      uint32_t code = cube_to_code(idx, L);
      atomicAdd(counts + tree * (int64_t(1) << (3 * L)) + code, 1u);
    }
  }
}

// ===========================================================================
// K2  pyramid: cube-order (or leaf-level path-order) bitsets -> path-order
//     per-level pyramids.  One CTA per (tree, chunk of <= 1024 leaf words).
// ===========================================================================
constexpr int PYR_BLOCK = 256;

// Leaf-level path-order word m (codes 32m..32m+31) from a cube bitset.
// Codes of one word share all but bits 0..4 = b0 g0 r0 b1 g1; the (b1,b0)
// quartet is 4 consecutive cube bits, so the word is 8 nibble gathers.
__device__ __forceinline__ uint32_t morton_word_from_cube(const uint32_t* __restrict__ cube, uint32_t m, int L) {
  if (L == 1) return cube[0] & 0xFFu;  // cube index == path code for L = 1
  const uint32_t base = code_to_cube(m << 5, L);
  uint32_t out = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const uint32_t g0 = c & 1, r0 = (c >> 1) & 1, g1 = (c >> 2) & 1;
    const uint32_t idx = base + ((g0 | (g1 << 1)) << L) + (r0 << (2 * L));
    const uint32_t nib = (cube[idx >> 5] >> (idx & 31u)) & 0xFu;
    const uint32_t sp = (nib & 3u) | ((nib & 12u) << 6);
    out |= sp << (g0 * 2 + r0 * 4 + g1 * 16);
  }
  return out;
}

template <bool FROM_CUBE>
__global__ void __launch_bounds__(PYR_BLOCK)
k_pyramid(const uint32_t* __restrict__ src, int64_t src_stride, int L, uint32_t* __restrict__ out) {
  __shared__ uint32_t s_w[PYR_CHUNK];
  __shared__ uint32_t s_c[PYR_CHUNK];
  const int64_t tree = blockIdx.y;
  const int64_t LW = level_words(L);
  const int64_t PW = pyr_words(L);
  const int64_t nw = LW < PYR_CHUNK ? LW : int64_t(PYR_CHUNK);        // words of this chunk at leaf level
  const int64_t w0 = int64_t(blockIdx.x) * nw;          // first leaf word of the chunk
  const uint32_t* s = src + tree * src_stride;
  uint32_t* o = out + tree * PW;
  // leaf level
  if (FROM_CUBE && L >= 5) {
    // The chunk is the level-(L-5) node w0/1024: a 32x32x32 sub-cube whose
    // 1024 (R', G') rows are one cube word each.  Stage them (and hand the
    // workspace back zeroed: each cube word belongs to exactly one chunk),
    // then gather 8 nibbles per path-order word.
    const uint32_t cb = code_to_cube(uint32_t(w0) << 5, L);
    const uint32_t M = (1u << L) - 1u;
    const uint32_t Rb = (cb >> (2 * L)) & M, Gb = (cb >> L) & M, Bw = (cb & M) >> 5;
    for (int t = threadIdx.x; t < PYR_CHUNK; t += PYR_BLOCK) {
      const uint32_t r = t >> 5, g = t & 31;
      uint32_t* cw = const_cast<uint32_t*>(s) + ((int64_t(Rb + r) << (2 * L - 5)) | (int64_t(Gb + g) << (L - 5)) | Bw);
      s_c[t] = *cw;
      if (s_c[t]) *cw = 0u;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < PYR_CHUNK; i += PYR_BLOCK) {
      const uint32_t c = uint32_t(i) << 5;
      const uint32_t rl = compact3(c >> 2), gl = compact3(c >> 1), bl = compact3(c);
      uint32_t x = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t g0 = k & 1, r0 = (k >> 1) & 1, g1 = (k >> 2) & 1;
        const uint32_t nib = (s_c[((rl + r0) << 5) + gl + g0 + 2 * g1] >> bl) & 0xFu;
        x |= ((nib & 3u) | ((nib & 12u) << 6)) << (g0 * 2 + r0 * 4 + g1 * 16);
      }
      s_w[i] = x;
      o[level_offset(L) + w0 + i] = x;          // the chunk owns these words
    }
  } else {
    for (int i = threadIdx.x; i < nw; i += PYR_BLOCK) {
      uint32_t x;
      if constexpr (FROM_CUBE) x = morton_word_from_cube(s, uint32_t(w0 + i), L);
      else x = s[w0 + i];
      if (L == 1) x &= 0xFFu;
      s_w[i] = x;
      o[level_offset(L) + w0 + i] = x;          // the chunk owns these words
    }
    if constexpr (FROM_CUBE) {                  // one chunk = the whole (small) tree
      __syncthreads();
      for (int i = threadIdx.x; i < cube_words(L); i += PYR_BLOCK) const_cast<uint32_t*>(s)[i] = 0u;
    }
  }
  __syncthreads();
  // bit range of the chunk at the current level: [B, B + n)
  int64_t B = w0 * 32, n = (L == 1) ? 8 : nw * 32;
  for (int l = L - 1; l >= 1; --l) {
    const int64_t off = level_offset(l);
    if (n >= 256) {            // parent range is whole words, owned by this CTA
      const int64_t pn = n / 256;
      uint32_t vals[PYR_CHUNK / 8 / PYR_BLOCK + 1];
      int cnt = 0;
      for (int64_t k = threadIdx.x; k < pn; k += PYR_BLOCK) {
        uint32_t v = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) v |= nz4(s_w[8 * k + q]) << (4 * q);
        vals[cnt++] = v;
      }
      __syncthreads();
      cnt = 0;
      for (int64_t k = threadIdx.x; k < pn; k += PYR_BLOCK) {
        const uint32_t v = vals[cnt++];
        s_w[k] = v;
        o[off + B / 256 + k] = v;               // owned: plain store, zeros included
      }
      __syncthreads();
      B /= 8;
      n /= 8;
    } else {                   // < 32 parent bits: one partial word, shared
      if (threadIdx.x == 0) {
        uint32_t v = 0;
        if (n >= 32) {
          for (int q = 0; q < n / 32; ++q) v |= nz4(s_w[q]) << (4 * q);
        } else {
          const uint32_t x = s_w[0];
          if (n >= 8) {
            for (int q = 0; q < n / 8; ++q) v |= (((x >> (8 * q)) & 0xFFu) != 0u) << q;
          } else {
            v = (x & ((1u << n) - 1u)) != 0u;
          }
        }
        s_w[0] = v;
      }
      __syncthreads();
      const int64_t pB = B / 8;
      const int64_t pn = n >= 8 ? n / 8 : 1;
      const uint32_t v = s_w[0];
      if (threadIdx.x == 0 && v) atomicOr(o + off + pB / 32, v << (pB % 32));
      __syncthreads();
      B = pB;
      n = pn;
    }
  }
}

// ===========================================================================
// K3  merge: per-node counts over trees, threshold k_min
// ===========================================================================
// One thread per (region, pyramid word).  Per-bit tree counts are kept as
// SWAR byte counters (acc[q] byte j counts bit q + 8j: 16 ops per tree and
// word), folded into 32-bit counters every 255 trees.  Loads are coalesced
// across threads (consecutive words of one tree).

// Merged leaf word m (path-code order) -> OR its 32 bits into the cube-order
// classify operand: the inverse of morton_word_from_cube (8 nibbles).
__device__ __forceinline__ void scatter_leaf_word_to_cube(uint32_t word, uint32_t m, int L, uint32_t* cube) {
  if (!word) return;
  if (L == 1) { atomicOr(cube, word & 0xFFu); return; }
  const uint32_t base = code_to_cube(m << 5, L);
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const uint32_t g0 = c & 1, r0 = (c >> 1) & 1, g1 = (c >> 2) & 1;
    const int off = g0 * 2 + r0 * 4 + g1 * 16;
    const uint32_t nib = ((word >> off) & 3u) | (((word >> (off + 8)) & 3u) << 2);
    if (nib) {
      const uint32_t idx = base + ((g0 | (g1 << 1)) << L) + (r0 << (2 * L));
      atomicOr(cube + (idx >> 5), nib << (idx & 31u));
    }
  }
}

__device__ __forceinline__ void finish_word(const uint32_t (&c32)[32], int64_t wi, int64_t w, int64_t r,
                                            int64_t k_min, int L, int64_t leaf_off, int64_t CW,
                                            uint32_t* counts, uint32_t* out, uint32_t* cube) {
  if (counts) {
    uint4* dst = reinterpret_cast<uint4*>(counts + wi * 32);
#pragma unroll
    for (int q = 0; q < 8; ++q) dst[q] = make_uint4(c32[4 * q], c32[4 * q + 1], c32[4 * q + 2], c32[4 * q + 3]);
  }
  if (out) {
    uint32_t bits = 0;
#pragma unroll
    for (int b = 0; b < 32; ++b) bits |= uint32_t(int64_t(c32[b]) >= k_min) << b;
    out[wi] = bits;
    if (cube && w >= leaf_off) scatter_leaf_word_to_cube(bits, uint32_t(w - leaf_off), L, cube + r * operand_words(L));
  }
}

// Block = 32 words (threadIdx.x, coalesced loads) x 8 tree groups
// (threadIdx.y): thread (x, y) counts trees y, y+8, ... of word x with SWAR
// byte counters, so each thread keeps <= ceil(n/8) independent loads in
// flight.  Groups are combined in shared memory; more than 255 trees per
// thread spill into 32-bit shared counters.
constexpr int MERGE_GROUPS = 8;
__global__ void __launch_bounds__(32 * MERGE_GROUPS)
k_merge(const uint32_t* __restrict__ pyr, int n_trees, int n_regions, int L, int64_t k_min,
        uint32_t* __restrict__ counts, uint32_t* __restrict__ out, uint32_t* __restrict__ cube) {
  __shared__ uint32_t s_acc[MERGE_GROUPS][8][32];
  __shared__ uint32_t s_wide[32][33];
  __shared__ uint32_t s_bits[MERGE_GROUPS][32];
  const int x = threadIdx.x, y = threadIdx.y;
  const int64_t PW = pyr_words(L);
  const int64_t total = PW * n_regions;
  const int64_t leaf_off = level_offset(L), CW = cube_words(L);
  const bool wide = (n_trees + MERGE_GROUPS - 1) / MERGE_GROUPS >= 252;   // a thread may flush
  for (int64_t base = int64_t(blockIdx.x) * 32; base < total; base += int64_t(gridDim.x) * 32) {
    const int64_t wi = base + x;
    const bool valid = wi < total;
    if (wide) {
      for (int i = y * 32 + x; i < 32 * 33; i += 32 * MERGE_GROUPS) (&s_wide[0][0])[i] = 0;
      __syncthreads();
    }
    uint32_t acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0;
    int since = 0;
    if (valid) {
      const uint32_t* p = pyr + wi;
      int t = y;
      for (; t + 3 * MERGE_GROUPS < n_trees; t += 4 * MERGE_GROUPS) {
        const uint32_t a = __ldg(p + int64_t(t) * total), b = __ldg(p + int64_t(t + MERGE_GROUPS) * total);
        const uint32_t d = __ldg(p + int64_t(t + 2 * MERGE_GROUPS) * total);
        const uint32_t e = __ldg(p + int64_t(t + 3 * MERGE_GROUPS) * total);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          acc[q] += ((a >> q) & 0x01010101u) + ((b >> q) & 0x01010101u) + ((d >> q) & 0x01010101u) +
                    ((e >> q) & 0x01010101u);
        since += 4;
        if (since > 251) {   // keep byte counters below 256
#pragma unroll
          for (int q = 0; q < 8; ++q) {
#pragma unroll
            for (int j = 0; j < 4; ++j) atomicAdd(&s_wide[x][q + 8 * j], (acc[q] >> (8 * j)) & 0xFFu);
            acc[q] = 0;
          }
          since = 0;
        }
      }
      for (; t < n_trees; t += MERGE_GROUPS) {
        const uint32_t a = __ldg(p + int64_t(t) * total);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] += (a >> q) & 0x01010101u;
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) s_acc[y][q][x] = acc[q];
    __syncthreads();
    // thread (x, y) totals bits y, y+8, y+16, y+24 of word x
    uint32_t c[4] = {0, 0, 0, 0};
#pragma unroll
    for (int g = 0; g < MERGE_GROUPS; ++g) {
      const uint32_t v = s_acc[g][y][x];
#pragma unroll
      for (int j = 0; j < 4; ++j) c[j] += (v >> (8 * j)) & 0xFFu;
    }
    if (wide) {
#pragma unroll
      for (int j = 0; j < 4; ++j) c[j] += s_wide[x][y + 8 * j];
    }
    uint32_t part = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) part |= uint32_t(int64_t(c[j]) >= k_min) << (y + 8 * j);
    s_bits[y][x] = part;
    if (valid && counts) {
#pragma unroll
      for (int j = 0; j < 4; ++j) counts[wi * 32 + y + 8 * j] = c[j];
    }
    __syncthreads();
    if (y == 0 && valid && out) {
      uint32_t bits = 0;
#pragma unroll
      for (int g = 0; g < MERGE_GROUPS; ++g) bits |= s_bits[g][x];
      out[wi] = bits;
      const int64_t r = wi / PW, w = wi - r * PW;
      if (cube && w >= leaf_off) scatter_leaf_word_to_cube(bits, uint32_t(w - leaf_off), L, cube + r * operand_words(L));
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Whole-model build (obg_build_model) in cube order.  The merge counts nodes
// per (level, cell) and does not care how a level's bits are ordered, so the
// per-tree levels stay in the cube order K1 produces: level l-1 from level l
// is an OR over 2x2x2 blocks -- four rows OR-ed, then adjacent bit pairs
// folded -- a few instructions per word instead of the 8 nibble gathers of
// a path-order word (k_pyramid: 12.9 us at C3, ncu r9).  Only the merged
// model (one tree per region) is converted to path order, and its leaf level
// is already the classify operand.
//   K1  k_build_flat   per tree: leaf cube + cube-order levels L-1..1 into
//                      the workspace (its flush; k_levels_cube when K1 has no
//                      shared bitset: L >= 7, generic grids)
//   K3f k_merge_fused  per node word: count over trees, threshold; merged
//                      leaf level -> the classify operand, every merged level
//                      -> the path-order pyramid (out_merged); workspace zeroed
// ---------------------------------------------------------------------------

// Levels L-1 .. 1 of tree t (cube order) into the workspace after its leaf
// cube, for the builds whose K1 has no shared-memory bitset (L >= 7, or the
// generic multi-region / unaligned path); one CTA per tree.  Levels of <= 8192 words (l <= 6) are staged in
// shared memory (ping-pong A/B), so the chain of levels costs one global
// round trip (the leaf load) instead of one per level (ncu r11: 10 us).
constexpr int LVL_BLOCK = 512;
constexpr uint32_t LVL_A = 8192, LVL_B = 1024;
__global__ void __launch_bounds__(LVL_BLOCK)
k_levels_cube(uint32_t* __restrict__ ws, int L) {
  __shared__ __align__(16) uint32_t s_a[LVL_A];
  __shared__ __align__(16) uint32_t s_b[LVL_B];
  const int64_t t = blockIdx.x;
  const uint32_t* leaf = ws + t * ws_words(L);
  uint32_t* o = ws + t * ws_words(L) + cube_words(L);   // upper levels, level_offset layout
  const uint32_t* child;
  uint32_t* cur = s_a;                             // smem buffer holding the child level (if staged)
  bool staged = false;
  if (L <= 6) {
    const uint32_t n = uint32_t(cube_words(L));
    if (n >= 4) {
      for (uint32_t i = threadIdx.x; i < n / 4; i += LVL_BLOCK)
        reinterpret_cast<uint4*>(s_a)[i] = __ldcg(reinterpret_cast<const uint4*>(leaf) + i);
    } else if (threadIdx.x < n) {
      s_a[threadIdx.x] = __ldcg(leaf + threadIdx.x);
    }
    __syncthreads();
    staged = true;
  }
  for (int l = L - 1; l >= 1; --l) {
    if (staged) child = cur;
    else child = (l == L - 1) ? leaf : o + level_offset(l + 1);
    uint32_t* parent = o + level_offset(l);
    uint32_t* next = (cur == s_a) ? s_b : s_a;
    const bool stage = l <= 6;                     // level fits the other buffer
    const uint32_t nw = uint32_t(level_words(l));
    for (uint32_t pw = threadIdx.x; pw < nw; pw += LVL_BLOCK) {
      const uint32_t v = reduce_cube_word(child, l, pw);
      parent[pw] = v;
      if (stage) (staged ? next : s_a)[pw] = v;
    }
    if (stage) {
      cur = staged ? next : s_a;
      staged = true;
    }
    __syncthreads();   // level l complete (and visible to the CTA) before level l-1 reads it
  }
}

// K3f block = 32 node words (threadIdx.x) x MERGE_GROUPS_C tree groups.
#ifndef OBG_MERGE_GROUPS
#define OBG_MERGE_GROUPS 16      // 4 trees per thread at C3: one round of loads (8 groups: +2-3 us)
#endif
constexpr int MERGE_GROUPS_C = OBG_MERGE_GROUPS;

// K3f: merge and path-order conversion in ONE launch (it replaced a merge
// kernel and a separate cube -> path-order kernel: two latency-bound launches
// of ~5 and ~4 us at C3).  Levels l >= 3 are cut into tiles of 2 R' x 4 G'
// rows (all B'): the 32 codes of a path-order word differ only in r0, g0, g1,
// b0, b1, so every path-order word lies inside one tile, and a CTA that
// merged a tile's cube words (tile-major, in shared memory) writes that
// tile's path-order words itself.  Levels 1..2 (3 words) are merged and
// converted by block 0 of each region.  Counting: 8 tree groups x 32 words,
// SWAR byte counters (bit q + 8j of a word in byte j of acc[q]), folded into
// 32-bit shared counters every 252 trees; the workspace is handed back zeroed.
// Count word `off` (relative to tree 0 of the region; off < 0: no word) over
// the trees of this thread's group and return the merged bits of the CTA's
// 32-word slot x (valid in thread y == 0).  Zeroes what it reads.
// MODE 0: merge (count + threshold); MODE 1: count only, the 32 per-bit
// counts of the slot's word written to counts_w[0..31] (a sharded build's
// partial counts, all-reduced across ranks); MODE 2: threshold counts_w
// (no tree loads).
template <int MODE>
__device__ __forceinline__ uint32_t merge_slot(uint32_t* __restrict__ ws, int64_t off, int64_t stride, int n_groups,
                                               int64_t k_min, uint32_t (&s_acc)[MERGE_GROUPS_C][8][32],
                                               uint32_t (&s_wide)[32][33], uint32_t (&s_bits)[8][32], bool wide,
                                               uint32_t* __restrict__ counts_w) {
  const int x = threadIdx.x, y = threadIdx.y;
  if constexpr (MODE == 2) {
    // counts of word x: bits from 32 u32 counts (one thread per word)
    uint32_t bits = 0;
    if (y == 0 && off >= 0) {
      const uint4* src = reinterpret_cast<const uint4*>(counts_w);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint4 v = __ldcg(src + q);
        bits |= (uint32_t(int64_t(v.x) >= k_min) << (4 * q)) | (uint32_t(int64_t(v.y) >= k_min) << (4 * q + 1)) |
                (uint32_t(int64_t(v.z) >= k_min) << (4 * q + 2)) | (uint32_t(int64_t(v.w) >= k_min) << (4 * q + 3));
      }
    }
    __syncthreads();
    return bits;
  }
  if (wide) {
    for (int i = y * 32 + x; i < 32 * 33; i += 32 * MERGE_GROUPS_C) (&s_wide[0][0])[i] = 0;
    __syncthreads();
  }
  uint32_t acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = 0;
  int since = 0;
  if (off >= 0) {
    uint32_t* p = ws + off;
    int t = y;
    for (; t + 3 * MERGE_GROUPS_C < n_groups; t += 4 * MERGE_GROUPS_C) {
      uint32_t* pa = p + int64_t(t) * stride;
      const int64_t st = int64_t(MERGE_GROUPS_C) * stride;
      const uint32_t a = __ldcg(pa), b = __ldcg(pa + st), d = __ldcg(pa + 2 * st), e = __ldcg(pa + 3 * st);
      if (a) pa[0] = 0u;
      if (b) pa[st] = 0u;
      if (d) pa[2 * st] = 0u;
      if (e) pa[3 * st] = 0u;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        acc[q] += ((a >> q) & 0x01010101u) + ((b >> q) & 0x01010101u) + ((d >> q) & 0x01010101u) +
                  ((e >> q) & 0x01010101u);
      since += 4;
      if (since > 251) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
#pragma unroll
          for (int j = 0; j < 4; ++j) atomicAdd(&s_wide[x][q + 8 * j], (acc[q] >> (8 * j)) & 0xFFu);
          acc[q] = 0;
        }
        since = 0;
      }
    }
    for (; t < n_groups; t += MERGE_GROUPS_C) {
      uint32_t* pa = p + int64_t(t) * stride;
      const uint32_t a = __ldcg(pa);
      if (a) *pa = 0u;
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] += (a >> q) & 0x01010101u;
    }
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) s_acc[y][q][x] = acc[q];
  __syncthreads();
  if (y < 8) {
    uint32_t c[4] = {0, 0, 0, 0};
#pragma unroll
    for (int g = 0; g < MERGE_GROUPS_C; ++g) {
      const uint32_t v = s_acc[g][y][x];
#pragma unroll
      for (int j = 0; j < 4; ++j) c[j] += (v >> (8 * j)) & 0xFFu;
    }
    if (wide) {
#pragma unroll
      for (int j = 0; j < 4; ++j) c[j] += s_wide[x][y + 8 * j];
    }
    if constexpr (MODE == 1) {
      if (off >= 0) {
#pragma unroll
        for (int j = 0; j < 4; ++j) counts_w[y + 8 * j] = c[j];
      }
    } else {
      uint32_t part = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) part |= uint32_t(int64_t(c[j]) >= k_min) << (y + 8 * j);
      s_bits[y][x] = part;
    }
  }
  __syncthreads();
  uint32_t bits = 0;
  if (MODE == 0 && y == 0) {
#pragma unroll
    for (int g = 0; g < 8; ++g) bits |= s_bits[g][x];
  }
  __syncthreads();                     // s_acc / s_bits are reused by the next slot
  return bits;
}

constexpr int MF_TOP = 2;              // levels 1..MF_TOP (3 words): block 0 of each region
constexpr int MF_TOP_WORDS = 3;        // pyr_words(2)

// Tile geometry of level l >= 3: words per tile WT = 2^(l-2) (8 rows of 2^l
// bits), tiles along G' = 2^(l-2); a block holds NWc = max(32, WT) slots.
__device__ __forceinline__ uint32_t mf_nwc(int l) { return l == 8 ? 64u : 32u; }
__host__ __device__ __forceinline__ int64_t mf_blocks(int l) {
  const int64_t n = level_words(l), c = l == 8 ? 64 : 32;
  return (n + c - 1) / c;
}
// cube word of tile t, tile-major slot jj (rows r0 = dr, dg = 0..3; B' fastest)
__device__ __forceinline__ uint32_t mf_tile_word(int l, uint32_t t, uint32_t jj) {
  const uint32_t gq_log = uint32_t(l - 2), WT = 1u << (l - 2);
  const uint32_t rp = t >> gq_log, gq = t & ((1u << gq_log) - 1u);
  const uint32_t half = WT >> 1;                                    // words per R' value
  const uint32_t dr = jj / half, q = jj % half;
  const uint32_t R = 2u * rp + dr;
  return ((((R << l) + 4u * gq) << l) >> 5) + q;                    // rows (R, 4gq..4gq+3) are contiguous
}

// counts (MODE 1 out / MODE 2 in): u32 [n_regions][PW][32], word w of the
// cube-order level layout (level_offset(l) + cube word), bit b at [w][b].
template <int MODE>
__global__ void __launch_bounds__(32 * MERGE_GROUPS_C)
k_merge_fused(uint32_t* __restrict__ ws, int n_groups, int n_regions, int L, int64_t k_min,
              uint32_t* __restrict__ cube, uint32_t* __restrict__ out, uint32_t* __restrict__ counts) {
  __shared__ uint32_t s_acc[MERGE_GROUPS_C][8][32];
  __shared__ uint32_t s_wide[32][33];
  __shared__ uint32_t s_bits[8][32];
  __shared__ uint32_t s_m[64];
  const int64_t r = blockIdx.y;
  const int x = threadIdx.x, y = threadIdx.y, tid = y * 32 + x;
  const int64_t PW = pyr_words(L), CW = cube_words(L), OW = operand_words(L), WSW = ws_words(L);
  const int64_t stride = WSW * n_regions;
  const bool wide = (n_groups + MERGE_GROUPS_C - 1) / MERGE_GROUPS_C >= 252;
  uint32_t* ws_r = ws + r * WSW;
  uint32_t* cube_r = cube + r * OW;
  uint32_t* out_r = out + r * PW;
  if (blockIdx.x == 0) {
    // levels 1..T (T <= 2): words 0 (level 1), 1..2 (level 2)
    const int T = L < MF_TOP ? L : MF_TOP;
    const int nw = int(level_offset(T + 1));
    const int w = x;
    int64_t off = -1;
    const int l = w == 0 ? 1 : 2;
    if (w < nw) off = (l == L) ? int64_t(w - level_offset(l)) : CW + w;
    uint32_t bits = merge_slot<MODE>(ws_r, off, stride, n_groups, k_min, s_acc, s_wide, s_bits, wide,
                                     counts + (r * PW + w) * 32);
    if constexpr (MODE == 1) return;
    if (y == 0 && w < nw) {
      if (l == 1) bits &= 0xFFu;
      s_m[w] = bits;
      if (l == L) cube_r[w - level_offset(l)] = bits;
    }
    __syncthreads();
    if (tid < nw) {
      const int lw = tid == 0 ? 1 : 2;
      const uint32_t m = uint32_t(tid - level_offset(lw));
      const uint32_t* lv = s_m + level_offset(lw);
      uint32_t word = 0;
      const int nb = lw == 1 ? 8 : 32;
      for (int bb = 0; bb < nb; ++bb) {
        const uint32_t idx = code_to_cube(m * 32u + uint32_t(bb), lw);
        word |= ((lv[idx >> 5] >> (idx & 31u)) & 1u) << bb;
      }
      out_r[tid] = word;
    }
    return;
  }
  // tile blocks: level l >= 3
  int64_t b = int64_t(blockIdx.x) - 1;
  int l = 3;
  for (; l <= L; ++l) {
    const int64_t nb = mf_blocks(l);
    if (b < nb) break;
    b -= nb;
  }
  if (l > L) return;
  const uint32_t WT = 1u << (l - 2);                               // words (and path words) per tile
  const uint32_t NWc = mf_nwc(l);
  const uint32_t gq_log = uint32_t(l - 2);
  const uint32_t LW = uint32_t(level_words(l));
  const uint32_t slot0 = uint32_t(b) * NWc;                        // first tile-major slot of the block
  const int64_t loff = level_offset(l);
  for (uint32_t pass = 0; pass < NWc / 32; ++pass) {
    const uint32_t j = pass * 32 + uint32_t(x);
    const uint32_t g = slot0 + j;                                  // global tile-major slot
    int64_t off = -1;
    uint32_t cw = 0;
    if (g < LW) {
      cw = mf_tile_word(l, g / WT, g % WT);
      off = (l == L) ? int64_t(cw) : CW + loff + cw;
    }
    const uint32_t bits = merge_slot<MODE>(ws_r, off, stride, n_groups, k_min, s_acc, s_wide, s_bits, wide,
                                           counts + (r * PW + loff + cw) * 32);
    if (MODE != 1 && y == 0 && g < LW) {
      s_m[j] = bits;
      if (l == L) cube_r[cw] = bits;
    }
  }
  if constexpr (MODE == 1) return;
  __syncthreads();
  if (uint32_t(tid) < NWc && slot0 + uint32_t(tid) < LW) {
    // path word: R>>1 = rp, G>>2 = gq, B>>2 = p; bit b0 + 2g0 + 4r0 + 8b1 + 16g1
    const uint32_t gs = slot0 + uint32_t(tid);
    const uint32_t t = gs / WT, p = gs % WT;
    const uint32_t rp = t >> gq_log, gq = t & ((1u << gq_log) - 1u);
    const uint32_t* tw = s_m + (t * WT - slot0);                    // the tile's words (tile-major)
    const uint32_t half = WT >> 1;
    uint32_t word = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint32_t g0 = c & 1, r0 = (c >> 1) & 1, g1 = (c >> 2) & 1;
      const uint32_t dg = g1 * 2u + g0;
      // bit of (B' = 4p) in row dg of the R'-half r0: rows are 2^l bits, the
      // half starts at its first row
      const uint32_t bit = (dg << l) + 4u * p;
      const uint32_t wv = tw[r0 * half + (bit >> 5)];
      const uint32_t nib = (wv >> (bit & 31u)) & 0xFu;
      word |= ((nib & 3u) | ((nib & 12u) << 6)) << (g0 * 2 + r0 * 4 + g1 * 16);
    }
    const uint32_t m = spread3(rp) | (spread3(p) << 1) | (spread3(gq) << 2);
    out_r[loff + m] = word;
  }
}

__global__ void __launch_bounds__(256)
k_threshold(const uint32_t* __restrict__ counts, int n_regions, int L, int64_t k_min, uint32_t* __restrict__ out,
            uint32_t* __restrict__ cube) {
  const int64_t PW = pyr_words(L);
  const int64_t total = PW * n_regions;
  const int64_t leaf_off = level_offset(L), CW = cube_words(L);
  for (int64_t wi = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; wi < total;
       wi += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = wi / PW, w = wi - r * PW;
    uint32_t c32[32];
    const uint4* src = reinterpret_cast<const uint4*>(counts + wi * 32);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint4 v = src[q];
      c32[4 * q] = v.x; c32[4 * q + 1] = v.y; c32[4 * q + 2] = v.z; c32[4 * q + 3] = v.w;
    }
    finish_word(c32, wi, w, r, k_min, L, leaf_off, CW, nullptr, out, cube);
  }
}

// ===========================================================================
// prune / leaf->cube
// ===========================================================================
// ---------------------------------------------------------------------------
// K3 (single-GPU model build, <= MC_MAX_TREES trees): bit-sliced merge and
// path-order conversion in one launch.  Four lanes per node word; a lane
// loads its share of the trees' words (up to 16 per round, all in flight)
// and compresses them with a Harley-Seal carry-save tree (15 full adders =
// 30 LOP3 per 16 words) into a 5-plane bit-sliced counter -- plane i holds
// bit i of the 32 per-bit-position tree counts; two shuffle + bit-sliced add
// steps give the word's counts, a borrow chain against k_min the merged
// word.  No shared-memory counters, one barrier (the path-order words of a
// tile are written by the CTA that merged it: CTAs own tiles of 2 R' x 4 G'
// cube rows, every 32-leaf path-order word lies inside one tile, as in
// k_merge_fused).  k_merge_fused (SWAR byte counters, 3 barriers per slot,
// ~12x the instructions) remains for > MC_MAX_TREES trees and for the
// sharded build's count / threshold modes.
// ---------------------------------------------------------------------------
#ifndef OBG_MERGE_CSA
#define OBG_MERGE_CSA 1
#endif
constexpr int MC_BLOCK = 256;                      // 64 node words per CTA
constexpr int MC_SLOTS = MC_BLOCK / 4;
constexpr int MC_MAX_TREES = 4 * 32;               // two rounds of 16 per lane

__device__ __forceinline__ uint32_t maj3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xE8;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ void csa(uint32_t& h, uint32_t& l, uint32_t a, uint32_t b, uint32_t c) {
  h = maj3(a, b, c);
  l = a ^ b ^ c;
}
// 16 words -> planes o[0..4] (counts 0..16)
__device__ __forceinline__ void harley_seal16(const uint32_t (&v)[16], uint32_t (&o)[5]) {
  uint32_t ones = 0, twos = 0, fours = 0, eights = 0, ta, tb, fa, fb, ea, eb;
  csa(ta, ones, ones, v[0], v[1]);   csa(tb, ones, ones, v[2], v[3]);   csa(fa, twos, twos, ta, tb);
  csa(ta, ones, ones, v[4], v[5]);   csa(tb, ones, ones, v[6], v[7]);   csa(fb, twos, twos, ta, tb);
  csa(ea, fours, fours, fa, fb);
  csa(ta, ones, ones, v[8], v[9]);   csa(tb, ones, ones, v[10], v[11]); csa(fa, twos, twos, ta, tb);
  csa(ta, ones, ones, v[12], v[13]); csa(tb, ones, ones, v[14], v[15]); csa(fb, twos, twos, ta, tb);
  csa(eb, fours, fours, fa, fb);
  uint32_t sixteens;
  csa(sixteens, eights, eights, ea, eb);
  o[0] = ones; o[1] = twos; o[2] = fours; o[3] = eights; o[4] = sixteens;
}

// Merged bits of ws word `w` (of region r) over n_groups trees; valid in lane
// sub == 0 of the four; every lane of the warp must call it.  Zeroes the
// words it reads (the workspace is handed back all-zero).
__device__ __forceinline__ uint32_t merge_word_csa(uint32_t* __restrict__ base, int64_t stride, int n_groups,
                                                   int64_t k_min, bool active, int sub) {
  uint32_t q[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int n_k = active ? (n_groups - sub + 3) / 4 : 0;         // trees sub, sub + 4, ...
  for (int k0 = 0; k0 < n_k; k0 += 16) {
    uint32_t v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j)
      v[j] = k0 + j < n_k ? __ldcg(base + int64_t(sub + 4 * (k0 + j)) * stride) : 0u;
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (v[j]) base[int64_t(sub + 4 * (k0 + j)) * stride] = 0u;
    uint32_t o[5];
    harley_seal16(v, o);
    uint32_t c = 0;                                                // q += o (bit-sliced)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t oi = i < 5 ? o[i] : 0u;
      const uint32_t s2 = q[i] ^ oi ^ c;
      c = maj3(q[i], oi, c);
      q[i] = s2;
    }
  }
#pragma unroll
  for (int step = 1; step <= 2; step <<= 1) {                      // + lanes sub ^ 1, then sub ^ 2
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t o = __shfl_xor_sync(0xFFFFFFFFu, q[i], step);
      const uint32_t s2 = q[i] ^ o ^ c;
      c = maj3(q[i], o, c);
      q[i] = s2;
    }
  }
  uint32_t borrow = 0;                                             // count >= k_min <=> no borrow
#pragma unroll
  for (int i = 0; i < 8; ++i) borrow = ((k_min >> i) & 1) ? (~q[i] | borrow) : (~q[i] & borrow);
  if ((k_min >> 8) != 0) borrow = 0xFFFFFFFFu;
  return ~borrow;
}

__global__ void __launch_bounds__(MC_BLOCK)
k_merge_tiles(uint32_t* __restrict__ ws, int n_groups, int n_regions, int L, int64_t k_min,
              uint32_t* __restrict__ cube, uint32_t* __restrict__ out) {
  __shared__ uint32_t s_m[MC_SLOTS];
  const int64_t r = blockIdx.y;
  const int64_t PW = pyr_words(L), CW = cube_words(L), OW = operand_words(L), WSW = ws_words(L);
  const int64_t stride = WSW * n_regions;
  const int tid = threadIdx.x, sub = tid & 3, j = tid >> 2;
  pdl_wait();                                        // the build kernel's workspace is complete
  pdl_launch_dependents();                           // a dependent classify may place its CTAs
  uint32_t* ws_r = ws + r * WSW;
  uint32_t* cube_r = cube + r * OW;
  uint32_t* out_r = out + r * PW;
  if (blockIdx.x == 0) {
    // levels 1..min(L, 2): words 0 (level 1), 1..2 (level 2)
    const int T = L < 2 ? L : 2;
    const int nw = int(level_offset(T + 1));
    const int l = j == 0 ? 1 : 2;
    const bool active = j < nw;
    const int64_t off = !active ? 0 : (l == L ? int64_t(j - level_offset(l)) : CW + j);
    uint32_t bits = merge_word_csa(ws_r + off, stride, n_groups, k_min, active, sub);
    if (active && sub == 0) {
      if (l == 1) bits &= 0xFFu;
      s_m[j] = bits;
      if (l == L) cube_r[j - level_offset(l)] = bits;
    }
    __syncthreads();
    if (tid < nw) {
      const int lw = tid == 0 ? 1 : 2;
      const uint32_t m = uint32_t(tid - level_offset(lw));
      const uint32_t* lv = s_m + level_offset(lw);
      uint32_t word = 0;
      const int nb = lw == 1 ? 8 : 32;
      for (int bb = 0; bb < nb; ++bb) {
        const uint32_t idx = code_to_cube(m * 32u + uint32_t(bb), lw);
        word |= ((lv[idx >> 5] >> (idx & 31u)) & 1u) << bb;
      }
      out_r[tid] = word;
    }
    return;
  }
  // tile blocks, level l >= 3: 64 tile-major slots per CTA
  int64_t b = int64_t(blockIdx.x) - 1;
  int l = 3;
  for (; l <= L; ++l) {
    const int64_t nb = (level_words(l) + MC_SLOTS - 1) / MC_SLOTS;
    if (b < nb) break;
    b -= nb;
  }
  if (l > L) return;
  const uint32_t WT = 1u << (l - 2);                               // words (and path words) per tile
  const uint32_t gq_log = uint32_t(l - 2);
  const uint32_t LW = uint32_t(level_words(l));
  const uint32_t slot0 = uint32_t(b) * MC_SLOTS;
  const int64_t loff = level_offset(l);
  const uint32_t g = slot0 + uint32_t(j);
  const bool active = g < LW;
  uint32_t cw = 0;
  if (active) cw = mf_tile_word(l, g / WT, g % WT);
  const int64_t off = (l == L) ? int64_t(cw) : CW + loff + cw;
  const uint32_t bits = merge_word_csa(ws_r + off, stride, n_groups, k_min, active, sub);
  if (active && sub == 0) {
    s_m[j] = bits;
    if (l == L) cube_r[cw] = bits;
  }
  __syncthreads();
  if (uint32_t(tid) < MC_SLOTS && slot0 + uint32_t(tid) < LW) {
    // path word: R>>1 = rp, G>>2 = gq, B>>2 = p; bit b0 + 2g0 + 4r0 + 8b1 + 16g1
    const uint32_t gs = slot0 + uint32_t(tid);
    const uint32_t t = gs / WT, p = gs % WT;
    const uint32_t rp = t >> gq_log, gq = t & ((1u << gq_log) - 1u);
    const uint32_t* tw = s_m + (t * WT - slot0);                    // the tile's words (tile-major)
    const uint32_t half = WT >> 1;
    uint32_t word = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint32_t g0 = c & 1, r0 = (c >> 1) & 1, g1 = (c >> 2) & 1;
      const uint32_t dg = g1 * 2u + g0;
      const uint32_t bit = (dg << l) + 4u * p;
      const uint32_t wv = tw[r0 * half + (bit >> 5)];
      const uint32_t nib = (wv >> (bit & 31u)) & 0xFu;
      word |= ((nib & 3u) | ((nib & 12u) << 6)) << (g0 * 2 + r0 * 4 + g1 * 16);
    }
    out_r[loff + (spread3(rp) | (spread3(p) << 1) | (spread3(gq) << 2))] = word;
  }
}

__global__ void k_prune(const uint32_t* __restrict__ pyr, int64_t PW, int64_t PW2, int64_t n_trees,
                        uint32_t* __restrict__ out) {
  const int64_t total = PW2 * n_trees;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = i / PW2, w = i - t * PW2;
    out[i] = pyr[t * PW + w];
  }
}

__global__ void k_leaf_cube(const uint32_t* __restrict__ pyr, int64_t PW, int L, int64_t n_trees,
                            uint32_t* __restrict__ cube) {
  const int64_t CW = cube_words(L);
  const int64_t off = level_offset(L);
  const int64_t total = CW * n_trees;
  const int nbits = L == 1 ? 8 : 32;   // writes the cube part of each region's operand
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = i / CW, cw = i - t * CW;
    const uint32_t* leaf = pyr + t * PW + off;
    uint32_t v = 0;
    for (int b = 0; b < nbits; ++b) {
      const uint32_t code = cube_to_code(uint32_t(cw * 32 + b), L);
      v |= ((__ldg(leaf + (code >> 5)) >> (code & 31u)) & 1u) << b;
    }
    cube[t * operand_words(L) + cw] = v;
  }
}

// L = 7 classify operand: 2-bit state per L=6 cell from the finished cube
// (some / all of its 8 leaves present), canonical order i = R6*256 + G6*4 + B6/16,
// stored after the cube.  State word = SWAR over the 4 cube words of rows
// (2R6+{0,1}, 2G6+{0,1}): bit pairs (2b, 2b+1) are the children along B'.
// One CTA (1024 threads) per region; also counts the mixed / occupied cells.
__global__ void __launch_bounds__(1024) k_l7_states(uint32_t* __restrict__ operand) {
  __shared__ uint32_t s_red[2][32];
  uint32_t* op = operand + int64_t(blockIdx.x) * operand_words(7);
  uint32_t mixed = 0, some = 0;
  // one thread per full-cell word = two state words (B6 = 0..15 | 16..31 of a half row)
  for (uint32_t j = threadIdx.x; j < uint32_t(S7_CELL_WORDS); j += 1024) {
    uint32_t cells = 0;
#pragma unroll
    for (uint32_t hq = 0; hq < 2; ++hq) {
      const uint32_t i = 2u * j + hq;
      const uint32_t r6 = i >> 8, g6 = (i >> 2) & 63u, q = i & 3u;
      const uint32_t b = (2u * r6) * 512u + (2u * g6) * 4u + q;
      const uint32_t w00 = op[b], w01 = op[b + 4], w10 = op[b + 512], w11 = op[b + 516];
      const uint32_t a = w00 | w01 | w10 | w11, A = w00 & w01 & w10 & w11;
      const uint32_t sm = (a | (a >> 1)) & 0x55555555u, al = (A & (A >> 1)) & 0x55555555u;
      op[cube_words(7) + i] = sm | (al << 1);
      some += __popc(sm);
      mixed += __popc(sm & ~al);
      uint32_t x = al;                                           // even bits -> low 16 bits
      x = (x | (x >> 1)) & 0x33333333u;
      x = (x | (x >> 2)) & 0x0F0F0F0Fu;
      x = (x | (x >> 4)) & 0x00FF00FFu;
      x = (x | (x >> 8)) & 0x0000FFFFu;
      cells |= x << (16u * hq);
    }
    op[S7_CELLS_OFF + j] = cells;                                // L=6 cube word (R6 << 7 | G6 << 1 | B6 >> 5)
  }
  mixed = __reduce_add_sync(0xFFFFFFFFu, mixed);
  some = __reduce_add_sync(0xFFFFFFFFu, some);
  if ((threadIdx.x & 31) == 0) {
    s_red[0][threadIdx.x >> 5] = mixed;
    s_red[1][threadIdx.x >> 5] = some;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    mixed = __reduce_add_sync(0xFFFFFFFFu, s_red[0][threadIdx.x]);
    some = __reduce_add_sync(0xFFFFFFFFu, s_red[1][threadIdx.x]);
    // the operand's 32-word tail: [0] mixed, [1] occupied, the rest zero
    op[S7_COUNTS_OFF + threadIdx.x] = threadIdx.x == 0 ? mixed : threadIdx.x == 1 ? some : 0u;
  }
}

// ===========================================================================
// K4  classify
// ===========================================================================
#ifndef OBG_CLS_BLOCK
#define OBG_CLS_BLOCK 256
#endif
constexpr int CLS_BLOCK = OBG_CLS_BLOCK;

// Flat path: 1x1 grid, leaf cube bitset in shared memory (L <= 6) or read
// through L1/L2 (L >= 7).  One thread = one 16-pixel unit per iteration:
// 3 x 16-byte loads, 16 lookups, one 16-byte (u8) or 2-byte (packed) store.

// What the classify kernels do with a unit's 16 presence bits: write the
// foreground mask (u8 or bit-packed), or -- fused evaluation, SURVEY.md
// §8(f) row 3 / evaluation.py:38-53 -- compare with a ground-truth mask and
// count the confusion (tn, tp, fn, fp) without writing any mask.
enum { OUT_U8 = 0, OUT_PACKED = 1, OUT_CONF_U8 = 2, OUT_CONF_PACKED = 3 };
struct ConfAcc {
  uint32_t tn = 0, tp = 0, fn = 0, fp = 0;
  __device__ __forceinline__ void add(uint32_t fg, uint32_t t, uint32_t valid) {
    tp += __popc(fg & t & valid);
    fp += __popc(fg & ~t & valid);
    fn += __popc(~fg & t & valid);
    tn += __popc(~fg & ~t & valid);
  }
};

// nonzero bytes of x -> bits 0..3
__device__ __forceinline__ uint32_t nz_nibble(uint32_t x) {
  const uint32_t hi = (((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x) & 0x80808080u;
  return ((hi >> 7) * 0x01020408u) >> 24;
}

// Presence bits (bit 0 of v[j]) of a 16-pixel unit -> 16 foreground mask
// bytes (one 16-byte streaming store) or 16 mask bits.
template <bool PACKED>
__device__ __forceinline__ void store_mask16(const uint32_t (&v)[16], uint8_t* mask, int64_t u) {
  if constexpr (!PACKED) {
    uint4 o;
    o.x = __byte_perm(__byte_perm(v[0], v[1], 0x0040), __byte_perm(v[2], v[3], 0x0040), 0x5410);
    o.y = __byte_perm(__byte_perm(v[4], v[5], 0x0040), __byte_perm(v[6], v[7], 0x0040), 0x5410);
    o.z = __byte_perm(__byte_perm(v[8], v[9], 0x0040), __byte_perm(v[10], v[11], 0x0040), 0x5410);
    o.w = __byte_perm(__byte_perm(v[12], v[13], 0x0040), __byte_perm(v[14], v[15], 0x0040), 0x5410);
    o.x = ~o.x & 0x01010101u; o.y = ~o.y & 0x01010101u;
    o.z = ~o.z & 0x01010101u; o.w = ~o.w & 0x01010101u;
    __stcs(reinterpret_cast<uint4*>(mask) + u, o);
  } else {
    uint32_t b = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) b |= (v[j] & 1u) << j;
    reinterpret_cast<uint16_t*>(mask)[u] = uint16_t(~b & 0xFFFFu);
  }
}

template <int OUT>
__device__ __forceinline__ void emit16(const uint32_t (&v)[16], uint8_t* out, int64_t u, ConfAcc& acc) {
  if constexpr (OUT == OUT_U8 || OUT == OUT_PACKED) {
    store_mask16<OUT == OUT_PACKED>(v, out, u);
  } else {
    uint32_t bg = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) bg |= (v[j] & 1u) << j;
    uint32_t t;
    if constexpr (OUT == OUT_CONF_U8) {
      const uint4 q = __ldcs(reinterpret_cast<const uint4*>(out) + u);
      t = nz_nibble(q.x) | (nz_nibble(q.y) << 4) | (nz_nibble(q.z) << 8) | (nz_nibble(q.w) << 12);
    } else {
      t = __ldcs(reinterpret_cast<const uint16_t*>(out) + u);
    }
    acc.add(~bg, t, 0xFFFFu);
  }
}

// single pixel i (tails): fg = 1 for foreground
template <int OUT>
__device__ __forceinline__ void emit1(uint32_t fg, uint8_t* out, int64_t i, ConfAcc& acc) {
  if constexpr (OUT == OUT_U8) out[i] = uint8_t(fg);
  else if constexpr (OUT == OUT_CONF_U8) acc.add(fg, out[i] != 0 ? 1u : 0u, 1u);
}

// block-end: warp sums, one 64-bit atomic per counter and warp
template <int OUT>
__device__ __forceinline__ void flush_conf(const ConfAcc& acc, unsigned long long* counts) {
  if constexpr (OUT == OUT_CONF_U8 || OUT == OUT_CONF_PACKED) {
    const uint32_t tn = __reduce_add_sync(0xFFFFFFFFu, acc.tn), tp = __reduce_add_sync(0xFFFFFFFFu, acc.tp);
    const uint32_t fn = __reduce_add_sync(0xFFFFFFFFu, acc.fn), fp = __reduce_add_sync(0xFFFFFFFFu, acc.fp);
    if ((threadIdx.x & 31) == 0) {
      if (tn) atomicAdd(counts + 0, (unsigned long long)tn);
      if (tp) atomicAdd(counts + 1, (unsigned long long)tp);
      if (fn) atomicAdd(counts + 2, (unsigned long long)fn);
      if (fp) atomicAdd(counts + 3, (unsigned long long)fp);
    }
  }
}

// One 16-pixel unit -> 16 mask bytes (or 16 mask bits).
template <int L, bool SMEM_BITS, int OUT>
__device__ __forceinline__ void classify_unit(const uint32_t (&w)[12], const uint32_t* bits, uint8_t* mask,
                                              int64_t u, ConfAcc& acc) {
  const char* base = reinterpret_cast<const char*>(bits);
  uint32_t v[16];
  if constexpr (SMEM_BITS) {
    // two pixels per address computation (see pair_positions)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      uint32_t aa, ba, ab, bb;
      pair_positions_dyn<SmemC<L>>(w, k, 0u, aa, ba, ab, bb);
      const uint32_t wa = *reinterpret_cast<const uint32_t*>(base + aa);
      const uint32_t wb = *reinterpret_cast<const uint32_t*>(base + ab);
      v[2 * k] = __funnelshift_r(wa, wa, ba);                       // bit 0 = background
      v[2 * k + 1] = __funnelshift_r(wb, wb, bb);
    }
  } else {
    uint32_t px[16];
    unpack16<0, L>(w, px);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      uint32_t addr, bsel;
      bit_position<L, SmemC<L>>(px[j], addr, bsel);
      const uint32_t wd = __ldg(reinterpret_cast<const uint32_t*>(base + addr));
      v[j] = __funnelshift_r(wd, wd, bsel);
    }
  }
  emit16<OUT>(v, mask, u, acc);
}

// `mask`: the output mask (OUT_U8 / OUT_PACKED) or the truth mask read by
// the fused evaluation (OUT_CONF_*, counts += tn, tp, fn, fp).
template <int L, bool SMEM_BITS, int OUT>
#ifndef OBG_CLS_MINB
#define OBG_CLS_MINB 2           // 4 CTAs per SM at L6; 5 or 6 (48 / 40 regs) lose L1 to shared memory: +3 % / +35 %
#endif
__global__ void __launch_bounds__(CLS_BLOCK, OBG_CLS_MINB)
k_classify_flat(const uint8_t* __restrict__ frames, int64_t n_units, int64_t n_pixels,
                const uint32_t* __restrict__ cube, uint8_t* __restrict__ mask, unsigned long long* counts,
                const uint32_t* __restrict__ gate) {
  // gate (L = 7 models classified through their L = 6 full-cell bitset):
  // the count of partly filled cells; this launch answers only when it is 0
  if (gate != nullptr && __ldg(gate) != 0u) return;
  ConfAcc acc;
  extern __shared__ uint32_t s_bits[];
  constexpr int64_t CW = cube_words(L);
  const uint32_t* bits = cube;
  pdl_wait();                                        // OBG_MASK_AFTER_MODEL: the merge's operand is complete
  if constexpr (SMEM_BITS) {
    for (uint32_t i = threadIdx.x; i < SmemC<L>::compact; i += CLS_BLOCK) {
      const uint32_t p = SmemC<L>::compact_word(i);
      s_bits[p] = smem_word_from_cube<SmemC<L>>(cube, p);
    }
    __syncthreads();
    bits = s_bits;
  }
  const int64_t stride = int64_t(gridDim.x) * CLS_BLOCK;
  // two units per thread and iteration: six 16-byte loads in flight
  for (int64_t u = int64_t(blockIdx.x) * CLS_BLOCK + threadIdx.x; u < n_units; u += 2 * stride) {
    const bool second = u + stride < n_units;
    uint32_t wa[12], wb[12];
    load_unit(frames, u, wa);
    if (second) load_unit(frames, u + stride, wb);
    classify_unit<L, SMEM_BITS, OUT>(wa, bits, mask, u, acc);
    if (second) classify_unit<L, SMEM_BITS, OUT>(wb, bits, mask, u + stride, acc);
  }
  // tail pixels (n_pixels not a multiple of 16; u8 layouts only)
  if constexpr (OUT == OUT_U8 || OUT == OUT_CONF_U8) {
    if (blockIdx.x == 0) {
      for (int64_t i = n_units * 16 + threadIdx.x; i < n_pixels; i += CLS_BLOCK) {
        const uint32_t x = Smem<L>::skew ? gbr_word_scalar(frames + 3 * i) : rgb_word_scalar(frames + 3 * i);
        uint32_t addr, bsel;
        bit_position<L, SmemC<L>>(x, addr, bsel);
        const uint32_t* wp = reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(bits) + addr);
        const uint32_t wd = SMEM_BITS ? *wp : __ldg(wp);
        emit1<OUT>(((wd >> (bsel & 31u)) & 1u) ^ 1u, mask, i, acc);
      }
    }
  }
  flush_conf<OUT>(acc, counts);
}

// ---------------------------------------------------------------------------
// L = 7 classify.  The 2^21-bit leaf set (256 KB) does not fit shared memory,
// and random lookups through L1 serialise on cache-line tags (ncu/bench r1:
// 23 % of HBM on uniform-random frames; a 2-CTA cluster splitting the set
// over DSMEM was slower still).  Instead shared memory holds a 2-bit state
// per L=6 cell -- no / some / all of its 8 leaves present (64 KB, skewed
// rows) -- and only pixels in a "some" cell read their leaf bit from the
// cube in global memory.  Full and empty cells answer from shared memory.
// State word (R6, G6, B6/16) = SWAR over the 4 cube words of rows
// (2R6+{0,1}, 2G6+{0,1}): bit pairs (2b, 2b+1) are the children along B'.
// ---------------------------------------------------------------------------
#ifndef OBG_S7_BLOCK
#define OBG_S7_BLOCK 1024        // 2 CTAs per SM (66 KB state table each): 1024 threads, -12 % at uniform L7
#endif
#ifndef OBG_S7_MINB
#define OBG_S7_MINB 1
#endif
constexpr int S7_BLOCK = OBG_S7_BLOCK;
constexpr uint32_t S7_ROWW = 257;                          // 64 G6 x 4 words + pad
constexpr uint32_t S7_WORDS = 64 * S7_ROWW;

// x = [*, G, B, R] (s = 1): R6 = x>>26, G6 = x[10..15], B6 = x[18..23].
// Returns the cell's state in bits 0 (some) and 1 (all).
__device__ __forceinline__ uint32_t s7_state(const uint32_t* s_state, uint32_t x) {
  const uint32_t r6 = __umulhi(x, 1u << 6);                          // x >> 26
  const uint32_t c = (__umulhi(x, 1u << 26) & (63u << 4)) | (__umulhi(x, 1u << 12) & 0xCu);
  const uint32_t w = *reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(s_state) +
                                                          r6 * (S7_ROWW * 4u) + c);
  return __funnelshift_r(w, w, __umulhi(x, 1u << 15) & 0x1Eu);       // (B6 & 15) * 2
}

__device__ __forceinline__ uint32_t l7_leaf_bit(const uint32_t* __restrict__ cube, uint32_t x) {
  const uint32_t idx = ((x >> 25) << 14) | (((x >> 9) & 127u) << 7) | ((x >> 17) & 127u);
  return (__ldg(cube + (idx >> 5)) >> (idx & 31u)) & 1u;
}
// Leaf word of x = [*, G, B, R] rotated so that bit 0 is the pixel's leaf:
// byte offset R'<<11 | G'<<4 | (B'>>5)<<2 from three shifts and two LOP3s,
// bit B' & 31 = the low bits of x >> 17 (funnel shifts use them mod 32).
__device__ __forceinline__ uint32_t l7_leaf_word(const char* __restrict__ cube, uint32_t x) {
  const uint32_t off = ((x >> 14) & 0x3F800u) | ((x >> 5) & 0x7F0u) | ((x >> 20) & 0xCu);
  const uint32_t wd = __ldg(reinterpret_cast<const uint32_t*>(cube + off));
  return __funnelshift_r(wd, wd, x >> 17);
}

// `leaf_run` (warp-uniform): > 0 while the warp is in leaf mode -- its
// recent units had pixels in partially filled L6 cells, so the state lookups
// are skipped and every pixel reads its leaf word directly (~11 instead of
// ~28 instructions per pixel when every unit is mixed, e.g. a constant-colour
// scene).  It counts down and the warp retries the state table at 0.
constexpr int L7_LEAF_RUN = 32;
constexpr int L7_LEAF_LANES = 4;       // A/B: 4 lanes keeps C3-like scenes at L7 in leaf mode, uniform 2.7x faster

// l7_leaf_word, the load predicated on `pred` (0 without a memory access)
__device__ __forceinline__ uint32_t l7_leaf_word_if(const char* __restrict__ cube, uint32_t x, uint32_t pred) {
  const uint32_t off = ((x >> 14) & 0x3F800u) | ((x >> 5) & 0x7F0u) | ((x >> 20) & 0xCu);
  uint32_t wd = 0;
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p ld.global.nc.u32 %0, [%1];\n\t}"
               : "+r"(wd) : "l"(cube + off), "r"(pred));
  return __funnelshift_r(wd, wd, x >> 17);
}
// 16 background bits (bit j = pixel j's leaf present) -> the unit's output
template <int OUT>
__device__ __forceinline__ void emit_bits(uint32_t bg, uint8_t* out, int64_t u, ConfAcc& acc) {
  const uint32_t fg = ~bg & 0xFFFFu;
  if constexpr (OUT == OUT_U8) {
    uint4 o;                                    // nibble -> four 0/1 bytes: n * 0x00204081 & 0x01010101
    o.x = ((fg & 15u) * 0x00204081u) & 0x01010101u;
    o.y = (((fg >> 4) & 15u) * 0x00204081u) & 0x01010101u;
    o.z = (((fg >> 8) & 15u) * 0x00204081u) & 0x01010101u;
    o.w = ((fg >> 12) * 0x00204081u) & 0x01010101u;
    __stcs(reinterpret_cast<uint4*>(out) + u, o);
  } else if constexpr (OUT == OUT_PACKED) {
    reinterpret_cast<uint16_t*>(out)[u] = uint16_t(fg);
  } else {
    uint32_t t;
    if constexpr (OUT == OUT_CONF_U8) {
      const uint4 q = __ldcs(reinterpret_cast<const uint4*>(out) + u);
      t = nz_nibble(q.x) | (nz_nibble(q.y) << 4) | (nz_nibble(q.z) << 8) | (nz_nibble(q.w) << 12);
    } else {
      t = __ldcs(reinterpret_cast<const uint16_t*>(out) + u);
    }
    acc.add(fg, t, 0xFFFFu);
  }
}

// One 16-pixel unit at L = 7.  The per-pixel results are kept as BITS of
// three registers (some / all / background) and every pixel's [*, G, B, R]
// operand is re-extracted from the unit's words where it is used, so the
// live set is the two units of the double buffer plus a handful of words:
// no local-memory spills at the 64-register cap of 2 x 512 threads per SM
// (the earlier px[16] / v[16] arrays spilled 136-228 bytes per thread).
template <int OUT>
__device__ __forceinline__ void classify_unit_l7(const uint32_t (&w)[12], const uint32_t* s_state,
                                                 const uint32_t* __restrict__ cube, uint8_t* mask, int64_t u,
                                                 ConfAcc& acc, int& leaf_run) {
  const char* cb = reinterpret_cast<const char*>(cube);
  uint32_t bg = 0;
  if (leaf_run > 0) {
    --leaf_run;
    for16([&](auto jc) {
      constexpr int j = decltype(jc)::value;
      bg |= (l7_leaf_word(cb, pixel_word_gbr<j>(w)) & 1u) << j;
    });
    emit_bits<OUT>(bg, mask, u, acc);
    return;
  }
  uint32_t some = 0, all = 0;
  for16([&](auto jc) {
    constexpr int j = decltype(jc)::value;
    const uint32_t st = s7_state(s_state, pixel_word_gbr<j>(w));
    some |= (st & 1u) << j;
    all |= ((st >> 1) & 1u) << j;
  });
  const uint32_t mixed = some & ~all;                               // some but not all leaves
  bg = all;
  const uint32_t bal = __ballot_sync(__activemask(), mixed != 0u);
  if (bal) {
    // pixels in partially filled cells read their leaf word (predicated
    // loads: no traffic for the others)
    for16([&](auto jc) {
      constexpr int j = decltype(jc)::value;
      bg |= (l7_leaf_word_if(cb, pixel_word_gbr<j>(w), (mixed >> j) & 1u) & 1u) << j;
    });
    // leaf mode only where partial cells are common (several lanes met one):
    // with sparse partial cells (e.g. uniform-random frames and a nearly
    // full model) the state table answers almost every pixel
    if (__popc(bal) >= L7_LEAF_LANES) leaf_run = L7_LEAF_RUN;
  }
  emit_bits<OUT>(bg, mask, u, acc);
}

template <int OUT>
__device__ __forceinline__ void classify_l7_states(const uint8_t* __restrict__ frames, int64_t n_units, int64_t n_pixels,
                                                   const uint32_t* __restrict__ cube, uint8_t* __restrict__ mask,
                                                   ConfAcc& acc, uint32_t* s_state) {
  for (uint32_t i = threadIdx.x; i < 64u * 256u; i += S7_BLOCK)       // states follow the cube (k_l7_states)
    s_state[(i >> 8) * S7_ROWW + (i & 255u)] = __ldg(cube + cube_words(7) + i);
  __syncthreads();
  const int64_t stride = int64_t(gridDim.x) * S7_BLOCK;
  int leaf_run = 0;
  for (int64_t u = int64_t(blockIdx.x) * S7_BLOCK + threadIdx.x; u < n_units; u += 2 * stride) {
    const bool second = u + stride < n_units;
    uint32_t wa[12], wb[12];
    load_unit(frames, u, wa);
    if (second) load_unit(frames, u + stride, wb);
    classify_unit_l7<OUT>(wa, s_state, cube, mask, u, acc, leaf_run);
    if (second) classify_unit_l7<OUT>(wb, s_state, cube, mask, u + stride, acc, leaf_run);
  }
  if constexpr (OUT == OUT_U8 || OUT == OUT_CONF_U8) {
    if (blockIdx.x == 0) {
      for (int64_t i = n_units * 16 + threadIdx.x; i < n_pixels; i += S7_BLOCK) {
        const uint32_t x = gbr_word_scalar(frames + 3 * i);
        const uint32_t st = s7_state(s_state, x);
        const uint32_t bg = ((st ^ (st >> 1)) & 1u) ? l7_leaf_bit(cube, x) : (st >> 1) & 1u;
        emit1<OUT>(bg ^ 1u, mask, i, acc);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// L = 7 classify, cube in shared memory: 7/8 of the 256 KB leaf cube -- the
// slabs R' < 112, each 512 words + 1 pad word so R' varies the bank -- fill
// 225 KB of one 1024-thread CTA's shared memory; pixels with R' >= 112
// (R >= 224) read the remaining 32 KB from global memory, where it stays
// L1-resident.  One direct lookup per pixel whatever the model looks like:
// the state-table kernel (k_classify_l7) needs a random cube gather from
// L1/L2 for every pixel in a partially filled L6 cell, which a half-full
// model turns into 0.16 of HBM.
// ---------------------------------------------------------------------------
constexpr int C7_BLOCK = 1024;
#ifndef OBG_L7_PATH
#define OBG_L7_PATH 0            // 0: by the model's cell counts, 1: state table always, 2: cube always
#endif
constexpr uint32_t C7_SLAB = 513;                          // words per R' slab (128 G' x 4) + pad
constexpr uint32_t C7_ROWS = 112;                          // R' slabs held in shared memory
constexpr uint32_t C7_WORDS = C7_ROWS * C7_SLAB;           // 57456 words = 229824 bytes
constexpr uint32_t C7_X_LIMIT = C7_ROWS << 25;             // x = [*, G, B, R]: R' = x >> 25

// pixel x = [*, G, B, R]: the leaf word in shared memory (R' < 112) or in the
// global cube, rotated so that bit 0 is the pixel's leaf (B' & 31 = x >> 17)
__device__ __forceinline__ uint32_t c7_inrow(uint32_t x) {             // G' * 16 + (B' >> 5) * 4
  return ((x >> 5) & 0x7F0u) | ((x >> 20) & 0xCu);
}
__device__ __forceinline__ uint32_t c7_smem_word(const char* s_base, uint32_t x) {
  const uint32_t off = __umulhi(x, 1u << 7) * (C7_SLAB * 4u) + c7_inrow(x);
  const uint32_t wd = *reinterpret_cast<const uint32_t*>(s_base + off);
  return __funnelshift_r(wd, wd, x >> 17);
}
__device__ __forceinline__ uint32_t c7_global_word(const char* __restrict__ cube, uint32_t x) {
  const uint32_t wd = __ldg(reinterpret_cast<const uint32_t*>(cube + (((x >> 14) & 0x3F800u) | c7_inrow(x))));
  return __funnelshift_r(wd, wd, x >> 17);
}

template <int OUT>
__device__ __forceinline__ void classify_unit_c7(const uint32_t (&w)[12], const char* s_base,
                                                 const char* __restrict__ cube, uint8_t* mask, int64_t u,
                                                 ConfAcc& acc) {
  uint32_t far = 0;
  for16([&](auto jc) {
    constexpr int j = decltype(jc)::value;
    far |= uint32_t(pixel_word_gbr<j>(w) >= C7_X_LIMIT) << j;
  });
  uint32_t bg = 0;
  if (!__any_sync(__activemask(), far != 0u)) {
    for16([&](auto jc) {                                 // every pixel of the warp's units in shared memory
      constexpr int j = decltype(jc)::value;
      bg |= (c7_smem_word(s_base, pixel_word_gbr<j>(w)) & 1u) << j;
    });
  } else {
    for16([&](auto jc) {                                 // bright-red pixels read the cube's last 16 slabs
      constexpr int j = decltype(jc)::value;
      const uint32_t x = pixel_word_gbr<j>(w);
      const uint32_t v = ((far >> j) & 1u) ? c7_global_word(cube, x) : c7_smem_word(s_base, x);
      bg |= (v & 1u) << j;
    });
  }
  emit_bits<OUT>(bg, mask, u, acc);
}

template <int OUT>
__device__ __forceinline__ void classify_l7_cube(const uint8_t* __restrict__ frames, int64_t n_units, int64_t n_pixels,
                                                 const uint32_t* __restrict__ cube, uint8_t* __restrict__ mask,
                                                 ConfAcc& acc, uint32_t* s_cube) {
  {
    const uint4* src = reinterpret_cast<const uint4*>(cube);
    for (uint32_t i = threadIdx.x; i < C7_ROWS * 128u; i += C7_BLOCK) {   // 128 uint4 per slab
      const uint4 v = __ldg(src + i);
      uint32_t* d = s_cube + (i >> 7) * C7_SLAB + (i & 127u) * 4u;
      d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
    }
  }
  __syncthreads();
  const char* s_base = reinterpret_cast<const char*>(s_cube);
  const char* cb = reinterpret_cast<const char*>(cube);
  const int64_t stride = int64_t(gridDim.x) * C7_BLOCK;
  for (int64_t u = int64_t(blockIdx.x) * C7_BLOCK + threadIdx.x; u < n_units; u += 2 * stride) {
    const bool second = u + stride < n_units;
    uint32_t wa[12], wb[12];
    load_unit(frames, u, wa);
    if (second) load_unit(frames, u + stride, wb);
    classify_unit_c7<OUT>(wa, s_base, cb, mask, u, acc);
    if (second) classify_unit_c7<OUT>(wb, s_base, cb, mask, u + stride, acc);
  }
  if constexpr (OUT == OUT_U8 || OUT == OUT_CONF_U8) {
    if (blockIdx.x == 0) {
      for (int64_t i = n_units * 16 + threadIdx.x; i < n_pixels; i += C7_BLOCK) {
        const uint32_t x = gbr_word_scalar(frames + 3 * i);
        const uint32_t v = x < C7_X_LIMIT ? c7_smem_word(s_base, x) : c7_global_word(cb, x);
        emit1<OUT>((v & 1u) ^ 1u, mask, i, acc);
      }
    }
  }
}

// The model picks the path (counts from k_l7_states, read on the device, so
// the launches stay graph-capturable): both kernels are launched, each with
// its own shared-memory size, and the one not chosen exits at once.
//  * L6 cells almost all full or empty (mixed < 1/32 of the occupied): the
//    2-bit state table (66 KB, L1 left for the few gathers) answers almost
//    every pixel (C4 uniform, full model: 0.21 ms vs 0.36 ms, 32 4K frames);
//  * otherwise the cube in shared memory, one direct lookup per pixel (a
//    half-full model 0.96 -> 0.36 ms; C3-like scene at L7 0.15 -> 0.125 ms;
//    a 15 %-mixed model on uniform frames 0.47 -> 0.19 ms).
// 0: state table, 1: cube in shared memory, 2: no partly filled cell -- the
// L=6 kernel on the full-cell bitset answers (k_classify_flat<6> with a gate)
#ifndef OBG_L7_CELLS
#define OBG_L7_CELLS 1
#endif
__device__ __forceinline__ int l7_path(const uint32_t* __restrict__ operand) {
  const uint32_t mixed = __ldg(operand + S7_COUNTS_OFF);
  const uint32_t some = __ldg(operand + S7_COUNTS_OFF + 1);
  if (OBG_L7_PATH == 0 && OBG_L7_CELLS && mixed == 0) return 2;
  return (OBG_L7_PATH == 2 || (OBG_L7_PATH == 0 && 32u * mixed >= some && mixed > 0)) ? 1 : 0;
}
static_assert(S7_BLOCK == C7_BLOCK, "one block size for both L7 paths");
template <int OUT, bool DIRECT>
__global__ void __launch_bounds__(C7_BLOCK, 1)
k_classify_l7(const uint8_t* __restrict__ frames, int64_t n_units, int64_t n_pixels, const uint32_t* __restrict__ cube,
              uint8_t* __restrict__ mask, unsigned long long* counts) {
  if (l7_path(cube) != (DIRECT ? 1 : 0)) return;
  ConfAcc acc;
  extern __shared__ __align__(16) uint32_t s_dyn[];
  if constexpr (DIRECT) classify_l7_cube<OUT>(frames, n_units, n_pixels, cube, mask, acc, s_dyn);
  else classify_l7_states<OUT>(frames, n_units, n_pixels, cube, mask, acc, s_dyn);
  flush_conf<OUT>(acc, counts);
}

// Region grid (R x C > 1, model.py:61-75), L <= 6, W % 16 == 0: blockIdx.y =
// region row r (a band of rows, region_bounds); the CTA holds the C operands
// of the band in shared memory (row layout, OPW words apart) and streams the
// band's 16-pixel units.  A unit lies in one column region unless a column
// boundary cuts it (at most C-1 units per row): those take a per-pixel path.
#ifndef OBG_BAND_BLOCK
#define OBG_BAND_BLOCK 1024       // one CTA per SM holds the C operands; 1024 threads: 3x4 grid 177 -> 125 us
#endif
constexpr int BAND_BLOCK = OBG_BAND_BLOCK;
template <int L>
struct BandOp {
  static constexpr uint32_t OPW = (uint32_t(SmemC<L>::words) + 31u) & ~31u;   // words per region operand
};

// one unit of a band: column region (or per-pixel regions where a boundary
// cuts it), lookups in that region's shared operand, 16 mask bytes / bits
template <int L, int OUT>
__device__ __forceinline__ void band_unit(const uint32_t (&w)[12], int k, int64_t ubase, int W16, int C,
                                          const int* s_cb, const char* sb, uint8_t* mask, ConfAcc& acc) {
  using LY = SmemC<L>;
  constexpr uint32_t OPW = BandOp<L>::OPW;
  const int x0 = (k % W16) * 16;
  int c = 0;
  while (c + 1 < C && x0 >= s_cb[c + 1]) ++c;
  uint32_t v[16];
  if (x0 + 15 < s_cb[c + 1]) {
    const char* base = sb + c * (OPW * 4u);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      uint32_t aa, ba, ab, bb;
      pair_positions_dyn<LY>(w, kk, 0u, aa, ba, ab, bb);
      const uint32_t xa = *reinterpret_cast<const uint32_t*>(base + aa);
      const uint32_t xb = *reinterpret_cast<const uint32_t*>(base + ab);
      v[2 * kk] = __funnelshift_r(xa, xa, ba);
      v[2 * kk + 1] = __funnelshift_r(xb, xb, bb);
    }
  } else {
    // a column boundary cuts the unit: region per pixel
    uint32_t px[16];
    unpack16<0, L>(w, px);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      int cj = 0;
      while (cj + 1 < C && x0 + j >= s_cb[cj + 1]) ++cj;
      uint32_t addr, bsel;
      bit_position<L, LY>(px[j], addr, bsel);
      const uint32_t wd = *reinterpret_cast<const uint32_t*>(sb + cj * (OPW * 4u) + addr);
      v[j] = __funnelshift_r(wd, wd, bsel);
    }
  }
  emit16<OUT>(v, mask, ubase + k, acc);
}

template <int L, int OUT>
__global__ void __launch_bounds__(BAND_BLOCK)
k_classify_band(const uint8_t* __restrict__ frames, int n_frames, int H, int W, int R, int C,
                const uint32_t* __restrict__ cube, uint8_t* __restrict__ mask, unsigned long long* counts) {
  using LY = SmemC<L>;
  constexpr uint32_t OPW = BandOp<L>::OPW;
  extern __shared__ uint32_t s_ops[];
  __shared__ int s_cb[17];
  ConfAcc acc;
  const int r = blockIdx.y;
  const int y0 = int((int64_t(r) * H + R - 1) / R), y1 = int((int64_t(r + 1) * H + R - 1) / R);
  if (threadIdx.x <= C) s_cb[threadIdx.x] = int((int64_t(threadIdx.x) * W + C - 1) / C);
  for (uint32_t c = 0; c < uint32_t(C); ++c) {
    const uint32_t* src = cube + (int64_t(r) * C + c) * operand_words(L);
    for (uint32_t i = threadIdx.x; i < LY::compact; i += BAND_BLOCK) {
      const uint32_t p = LY::compact_word(i);
      s_ops[c * OPW + p] = smem_word_from_cube<LY>(src, p);
    }
  }
  __syncthreads();
  const int W16 = W / 16;
  const int64_t upf = int64_t(H) * W16;                         // units per frame
  const int band_units = (y1 - y0) * W16;
  const char* sb = reinterpret_cast<const char*>(s_ops);
  // the band's units of ALL frames as one index space, so the grid is sized
  // by the work (every SM busy) rather than by one frame's band
  const int64_t total = int64_t(band_units) * n_frames;
  const int64_t stride = int64_t(gridDim.x) * BAND_BLOCK;
  for (int64_t k = int64_t(blockIdx.x) * BAND_BLOCK + threadIdx.x; k < total; k += 2 * stride) {
    // two units per iteration: six 16-byte loads in flight
    uint32_t wa[12], wb[12];
    const int fa = int(k / band_units), ka = int(k - int64_t(fa) * band_units);
    const int64_t ubase_a = int64_t(fa) * upf + int64_t(y0) * W16;
    const bool second = k + stride < total;
    int kb = 0;
    int64_t ubase_b = 0;
    load_unit(frames, ubase_a + ka, wa);
    if (second) {
      const int fb = int((k + stride) / band_units);
      kb = int(k + stride - int64_t(fb) * band_units);
      ubase_b = int64_t(fb) * upf + int64_t(y0) * W16;
      load_unit(frames, ubase_b + kb, wb);
    }
    band_unit<L, OUT>(wa, ka, ubase_a, W16, C, s_cb, sb, mask, acc);
    if (second) band_unit<L, OUT>(wb, kb, ubase_b, W16, C, s_cb, sb, mask, acc);
  }
  flush_conf<OUT>(acc, counts);
}

template <int L, int OUT>
static int launch_classify_band(const uint8_t* frames, int n_frames, int H, int W, int R, int C, const uint32_t* cube,
                                uint8_t* mask, unsigned long long* counts, cudaStream_t st) {
  const size_t smem = size_t(C) * BandOp<L>::OPW * 4;
  static DevCache attr_smem;
  if (int(smem) > attr_smem()) {
    CUDA_TRY(cudaFuncSetAttribute(k_classify_band<L, OUT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr_smem() = int(smem);
  }
  const int bps = occupancy(k_classify_band<L, OUT>, BAND_BLOCK, smem);
  // R bands x per_band CTAs within one wave (rounding up would leave a
  // second wave of a few CTAs: 3 x 50 on 148 SMs doubled the 3x4 time)
  const int64_t per_band = std::max<int64_t>(1, int64_t(sm_count()) * bps / R);
  const int64_t band_units = (int64_t(H) / R + 1) * (W / 16);
  int64_t gx = min(per_band, (band_units * n_frames + BAND_BLOCK - 1) / BAND_BLOCK);
  if (gx < 1) gx = 1;
  k_classify_band<L, OUT><<<dim3(unsigned(gx), unsigned(R)), BAND_BLOCK, smem, st>>>(frames, n_frames, H, W, R, C, cube,
                                                                                    mask, counts);
  LAUNCH_CHECK("k_classify_band");
  return OBG_OK;
}

// Generic path: any grid / alignment / frame size.  One thread = 8 pixels of
// one frame (one packed byte, or 8 u8 mask bytes).
template <int OUT>
__global__ void __launch_bounds__(256)
k_classify_generic(const uint8_t* __restrict__ frames, int64_t n_frames, int H, int W, int L, int R, int C,
                   const uint32_t* __restrict__ cube, uint8_t* __restrict__ mask, unsigned long long* counts) {
  constexpr bool PACKED = OUT == OUT_PACKED || OUT == OUT_CONF_PACKED;
  ConfAcc acc;
  const int64_t P = int64_t(H) * W;
  const int64_t bytes_per_frame = (P + 7) / 8;
  const int64_t total = bytes_per_frame * n_frames;
  const int64_t CW = cube_words(L);
  const int s = 8 - L;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t f = t / bytes_per_frame, q = t - f * bytes_per_frame;
    uint32_t byte = 0;
    for (int k = 0; k < 8; ++k) {
      const int64_t p = q * 8 + k;
      if (p >= P) break;
      const int y = int(p / W), x = int(p - int64_t(y) * W);
      const int row = min(R - 1, int(int64_t(y) * R / H));
      const int col = min(C - 1, int(int64_t(x) * C / W));
      const uint8_t* px = frames + 3 * (f * P + p);
      const uint32_t idx = ((uint32_t(px[0]) >> s) << (2 * L)) | ((uint32_t(px[1]) >> s) << L) |
                           (uint32_t(px[2]) >> s);
      const uint32_t* bits = cube + (int64_t(row) * C + col) * operand_words(L);
      const uint32_t fg = ((__ldg(bits + (idx >> 5)) >> (idx & 31u)) & 1u) ^ 1u;
      if (PACKED) byte |= fg << k;
      else emit1<OUT>(fg, mask, f * P + p, acc);
    }
    if constexpr (OUT == OUT_PACKED) mask[t] = uint8_t(byte);
    if constexpr (OUT == OUT_CONF_PACKED) {
      const uint32_t nv = uint32_t(min(int64_t(8), P - q * 8));
      acc.add(byte, mask[t], (1u << nv) - 1u);
    }
  }
  flush_conf<OUT>(acc, counts);
}

// ===========================================================================
// pack_codes
// ===========================================================================
__global__ void k_pack_codes(const uint8_t* __restrict__ px, int64_t n, int L, uint32_t* __restrict__ codes) {
  const int sh = 3 * (8 - L);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const uint8_t* p = px + 3 * i;
    const uint32_t full = (spread3(p[0]) << 2) | (spread3(p[1]) << 1) | spread3(p[2]);
    codes[i] = full >> sh;
  }
}

// ===========================================================================
// serialize: preorder child-mask bytes from a pyramid
// ===========================================================================
// Preorder position of node (l, p) (l = 0 is the root):
//   pos = sum_{m<l} (rank_m(p >> 3(l-m)) + 1) + sum_{m>=l} rank_m(p << 3(m-l))
// where rank_m(q) = number of level-m nodes with code < q.  Node (l, p) emits
// byte p of level l+1 (its child mask), leaves emit 0 (octree.py:258-267).
// Exclusive popcount prefix over ALL words of the pyramid (levels
// concatenated), prefix[PW] = the node count, in two multi-CTA launches:
// per-chunk totals, then each CTA adds the totals of the chunks before it and
// scans its own chunk.  A level's local rank is prefix[off + w] - prefix[off].
constexpr int SCAN_BLOCK = 1024;
constexpr int SCAN_CHUNK = 4 * SCAN_BLOCK;       // words per CTA (4 per thread)

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* s_warp, uint32_t& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, x, d);
    if (lane >= d) x += t;
  }
  if (lane == 31) s_warp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t y = lane < SCAN_BLOCK / 32 ? s_warp[lane] : 0u;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, y, d);
      if (lane >= d) y += t;
    }
    s_warp[lane] = y;                                  // inclusive warp totals
  }
  __syncthreads();
  total = s_warp[SCAN_BLOCK / 32 - 1];
  const uint32_t before = wid ? s_warp[wid - 1] : 0u;
  __syncthreads();
  return before + x - v;
}

__global__ void __launch_bounds__(SCAN_BLOCK)
k_scan_partials(const uint32_t* __restrict__ pyr, int64_t PW, uint32_t* __restrict__ partials) {
  __shared__ uint32_t s_warp[32];
  const int64_t base = int64_t(blockIdx.x) * SCAN_CHUNK + 4 * threadIdx.x;
  uint32_t c = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) c += base + k < PW ? __popc(pyr[base + k]) : 0u;
  uint32_t total;
  block_exclusive_scan(c, s_warp, total);
  if (threadIdx.x == 0) partials[blockIdx.x] = total;
}

__global__ void __launch_bounds__(SCAN_BLOCK)
k_scan_finish(const uint32_t* __restrict__ pyr, int64_t PW, const uint32_t* __restrict__ partials,
              uint32_t* __restrict__ prefix) {
  __shared__ uint32_t s_warp[32];
  __shared__ uint32_t s_carry;
  if (threadIdx.x < 32) {
    uint32_t c = 0;
    for (uint32_t b = threadIdx.x; b < blockIdx.x; b += 32) c += partials[b];
    c = __reduce_add_sync(0xFFFFFFFFu, c);
    if (threadIdx.x == 0) s_carry = c;
  }
  const int64_t base = int64_t(blockIdx.x) * SCAN_CHUNK + 4 * threadIdx.x;
  uint32_t pc[4], c = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    pc[k] = base + k < PW ? __popc(pyr[base + k]) : 0u;
    c += pc[k];
  }
  uint32_t total;
  uint32_t run = block_exclusive_scan(c, s_warp, total) + s_carry;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (base + k < PW) prefix[base + k] = run;
    run += pc[k];
  }
  if (base <= PW && PW < base + 4) prefix[PW] = s_carry + total;   // the CTA holding the end writes the node count
  if (PW == int64_t(gridDim.x) * SCAN_CHUNK && blockIdx.x == gridDim.x - 1 && threadIdx.x == SCAN_BLOCK - 1)
    prefix[PW] = s_carry + total;
}

__device__ __forceinline__ uint32_t rank_of(const uint32_t* __restrict__ pyr, const uint32_t* __restrict__ prefix,
                                            int l, uint64_t q) {
  const int64_t off = level_offset(l);
  const uint64_t w = q >> 5;
  const uint32_t b = uint32_t(q & 31u);
  const uint32_t word = pyr[off + w];
  return prefix[off + w] - __ldg(prefix + off) + __popc(b ? (word & ((1u << b) - 1u)) : 0u);
}

// One thread per (pyramid word, bit): a warp shares one word, so the level
// search and the word load are warp-uniform, and each node's L rank lookups
// are independent loads (ILP) instead of a per-word serial loop over its bits.
__global__ void __launch_bounds__(256)
k_serialize(const uint32_t* __restrict__ pyr, const uint32_t* __restrict__ prefix, int L, uint8_t* __restrict__ out) {
  const int64_t PW = pyr_words(L);
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < PW * 32; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t gw = t >> 5;
    const int b = int(t & 31);
    const uint32_t word = __ldg(pyr + gw);
    if (!((word >> b) & 1u)) continue;
    int l = 1;
    while (l < L && gw >= level_offset(l + 1)) ++l;
    const int64_t w = gw - level_offset(l);
    const uint64_t p = uint64_t(w) * 32 + uint64_t(b);
    uint64_t pos = 1;  // the root precedes every node
    for (int m = 1; m < l; ++m) pos += rank_of(pyr, prefix, m, p >> (3 * (l - m))) + 1;
    for (int m = l; m <= L; ++m) pos += rank_of(pyr, prefix, m, p << (3 * (m - l)));
    uint8_t byte = 0;
    if (l < L) {
      const uint32_t cw = __ldg(pyr + level_offset(l + 1) + (p >> 2));
      byte = uint8_t(cw >> (8 * (p & 3)));
    }
    out[pos] = byte;
  }
}

// ===========================================================================
// Comparison baselines (reference detect.py:56-83):
// frame difference and the running-mean background, same masks (and the
// same IEEE binary64 running mean) as the reference's numpy code.
// ===========================================================================
// Frame difference: foreground iff some channel changed by strictly more than
// thr (detect.py:56-63).  Pair i = (prev + i*3P, cur + i*3P).  When cur ==
// prev + 3P (a sequence), a thread walks its unit position through a chunk
// of consecutive frames and keeps the previous unit in registers: 3 B read +
// 1 B written per pixel instead of 6 + 1.  Bytes: per-byte |c - p| > thr with
// SIMD byte ops, then OR of a pixel's three flags.
constexpr int FD_BLOCK = 256;

// flags (0x00 / 0xFF per byte) of the 12 words of a unit -> 16 mask bytes
__device__ __forceinline__ uint4 fd_mask16(const uint32_t (&f)[12]) {
  uint32_t o[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    // pixels 4q..4q+3 = bytes 12q..12q+11 = words 3q..3q+2
    // pixel k's three bytes land in byte k of x, y, z:
    // x = [a0 a3 b2 c1], y = [a1 b0 b3 c2], z = [a2 b1 c0 c3]
    const uint32_t a = f[3 * q], b = f[3 * q + 1], c = f[3 * q + 2];
    const uint32_t x = __byte_perm(__byte_perm(a, b, 0x0630), c, 0x5210);
    const uint32_t y = __byte_perm(__byte_perm(a, b, 0x0741), c, 0x6210);
    const uint32_t z = __byte_perm(__byte_perm(a, b, 0x0052), c, 0x7410);
    o[q] = (x | y | z) & 0x01010101u;
  }
  return make_uint4(o[0], o[1], o[2], o[3]);
}

__device__ __forceinline__ uint32_t fd_flags(uint32_t c, uint32_t p, uint32_t thr4) {
  return __vcmpgtu4(__vabsdiffu4(c, p), thr4);                     // 0xFF where |c - p| > thr
}

// mode: 0 = compare (thr in 0..254), 1 = all foreground (thr < 0), 2 = none (thr >= 255)
__global__ void __launch_bounds__(FD_BLOCK)
k_frame_diff(const uint8_t* __restrict__ prev, const uint8_t* __restrict__ cur, int n_pairs, int64_t pixels,
             int64_t n_units, int chunk, int thr, int mode, int seq, uint8_t* __restrict__ masks) {
  const int64_t fb = 3 * pixels;
  const int n_chunks = (n_pairs + chunk - 1) / chunk;
  const uint32_t thr4 = uint32_t(thr & 0xFF) * 0x01010101u;
  for (int64_t item = blockIdx.x * int64_t(FD_BLOCK) + threadIdx.x; item < n_units * n_chunks;
       item += int64_t(gridDim.x) * FD_BLOCK) {
    const int64_t u = item % n_units;
    const int i0 = int(item / n_units) * chunk, i1 = min(n_pairs, i0 + chunk);
    uint32_t wp[12], wc[12];
    if (mode == 0) load_unit(prev + int64_t(i0) * fb, u, wp);
    for (int i = i0; i < i1; ++i) {
      uint4 m;
      if (mode == 0) {
        if (!seq && i > i0) load_unit(prev + int64_t(i) * fb, u, wp);
        load_unit(cur + int64_t(i) * fb, u, wc);
        uint32_t f[12];
#pragma unroll
        for (int k = 0; k < 12; ++k) f[k] = fd_flags(wc[k], wp[k], thr4);
        m = fd_mask16(f);
        if (seq) {
#pragma unroll
          for (int k = 0; k < 12; ++k) wp[k] = wc[k];
        }
      } else {
        const uint32_t v = mode == 1 ? 0x01010101u : 0u;
        m = make_uint4(v, v, v, v);
      }
      __stcs(reinterpret_cast<uint4*>(masks + int64_t(i) * pixels) + u, m);
    }
  }
}

// generic path (pixels % 16 != 0 or unaligned buffers): one thread per pixel
__global__ void __launch_bounds__(FD_BLOCK)
k_frame_diff_px(const uint8_t* __restrict__ prev, const uint8_t* __restrict__ cur, int n_pairs, int64_t pixels,
                int thr, uint8_t* __restrict__ masks) {
  const int64_t total = int64_t(n_pairs) * pixels;
  for (int64_t k = blockIdx.x * int64_t(FD_BLOCK) + threadIdx.x; k < total; k += int64_t(gridDim.x) * FD_BLOCK) {
    const uint8_t* a = prev + 3 * k;
    const uint8_t* b = cur + 3 * k;
    int d = 0;
#pragma unroll
    for (int c = 0; c < 3; ++c) d = max(d, abs(int(b[c]) - int(a[c])));
    masks[k] = uint8_t(d > thr);
  }
}

// Running mean (detect.py:66-83): per pixel, for frames t = 0..n-1,
// mask = max_c |x_c - avg_c| > thr with the mean BEFORE the update (a NaN
// channel makes numpy's max NaN and the pixel background), then
// avg_c = avg_c + (x_c - avg_c) / (seen + t + 1): three correctly rounded
// binary64 operations in the reference's order (the quotient by div_by,
// correctly rounded), so the mean is bit-identical to numpy's.
// RN(d / n) from y = RN(1/n): q0 = RN(d y), r = d - n q0 (exact, one FMA),
// q = RN(q0 + r y) is the correctly rounded quotient (Markstein's theorem;
// checked against exact rational arithmetic on 300k cases, tools note in
// DESIGN.md).  Outside the normal range of d (tiny, huge, inf, NaN) the
// IEEE division is used.  3 FP64 ops instead of a ~10-op division sequence.
__device__ __forceinline__ double div_by(double d, double n, double y) {
  const double ad = fabs(d);
  if ((ad > 0x1p-900 && ad < 0x1p900) || d == 0.0) {
    const double q0 = __dmul_rn(d, y);
    const double r = __fma_rn(-q0, n, d);
    return __fma_rn(r, y, q0);
  }
  return __ddiv_rn(d, n);
}

__global__ void __launch_bounds__(FD_BLOCK)
k_running_average(const uint8_t* __restrict__ frames, int n_frames, int64_t pixels, int64_t seen,
                  double* __restrict__ average, double thr, uint8_t* __restrict__ masks) {
  for (int64_t p = blockIdx.x * int64_t(FD_BLOCK) + threadIdx.x; p < pixels; p += int64_t(gridDim.x) * FD_BLOCK) {
    double a0 = average[3 * p], a1 = average[3 * p + 1], a2 = average[3 * p + 2];
    constexpr int RA_UNROLL = 8;                                     // frames whose bytes are loaded up front
    for (int t0 = 0; t0 < n_frames; t0 += RA_UNROLL) {
      uint8_t xb[RA_UNROLL][3];
#pragma unroll
      for (int k = 0; k < RA_UNROLL; ++k) {
        if (t0 + k < n_frames) {
          const uint8_t* x = frames + (int64_t(t0 + k) * pixels + p) * 3;
          xb[k][0] = __ldcs(x); xb[k][1] = __ldcs(x + 1); xb[k][2] = __ldcs(x + 2);
        }
      }
#pragma unroll
      for (int k = 0; k < RA_UNROLL; ++k) {
        const int t = t0 + k;
        if (t >= n_frames) break;
        const double d0 = __dsub_rn(double(xb[k][0]), a0), d1 = __dsub_rn(double(xb[k][1]), a1),
                     d2 = __dsub_rn(double(xb[k][2]), a2);
        const double e0 = fabs(d0), e1 = fabs(d1), e2 = fabs(d2);
        const bool nan = (e0 != e0) | (e1 != e1) | (e2 != e2);
        masks[int64_t(t) * pixels + p] = uint8_t(!nan && ((e0 > thr) | (e1 > thr) | (e2 > thr)));
        const double n = double(seen + t + 1);
        const double y = __ddiv_rn(1.0, n);                          // RN(1/n), once per frame
        a0 = __dadd_rn(a0, div_by(d0, n, y));
        a1 = __dadd_rn(a1, div_by(d1, n, y));
        a2 = __dadd_rn(a2, div_by(d2, n, y));
      }
    }
    average[3 * p] = a0;
    average[3 * p + 1] = a1;
    average[3 * p + 2] = a2;
  }
}

// ===========================================================================
// C ABI
// ===========================================================================
static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static int grid_for(int64_t work, int block, int max_blocks) {
  int64_t g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > max_blocks) g = max_blocks;
  return int(g);
}

// C-ABI entry points: C linkage comes from the declarations in obg.h.

int obg_abi_version(void) { return OBG_ABI_VERSION; }
const char* obg_last_error(void) { return g_err; }

int64_t obg_pyramid_words(int levels) { return (levels < 1 || levels > 8) ? -1 : pyr_words(levels); }
int64_t obg_level_offset(int levels, int level) {
  if (levels < 1 || levels > 8 || level < 1 || level > levels) return -1;
  return level_offset(level);
}
int64_t obg_cube_words(int levels) { return (levels < 1 || levels > 8) ? -1 : operand_words(levels); }
int64_t obg_build_workspace_bytes(int n_trees, int n_regions, int levels) {
  if (levels < 1 || levels > 8 || n_trees < 0 || n_regions < 1) return -1;
  return int64_t(n_trees) * n_regions * ws_words(levels) * 4;
}

int obg_pack_codes(const uint8_t* pixels, int64_t n_pixels, int levels, uint32_t* codes, void* stream) {
  g_err[0] = 0;
  if (levels < 1 || levels > 8) return set_err(OBG_EINVAL, "levels must be in 1..8, got %d", levels);
  if (n_pixels < 0) return set_err(OBG_EINVAL, "n_pixels must be >= 0");
  if (n_pixels == 0) return OBG_OK;
  if (!pixels || !codes) return set_err(OBG_EINVAL, "null buffer");
  k_pack_codes<<<grid_for(n_pixels, 256, sm_count() * 16), 256, 0, as_stream(stream)>>>(pixels, n_pixels, levels, codes);
  LAUNCH_CHECK("k_pack_codes");
  return OBG_OK;
}

#ifndef OBG_BYTE_TABLE
#define OBG_BYTE_TABLE 1
#endif
// Units per CTA of the segment-streaming kernels (K1 flat / byte table /
// L7 halves / histogram): the CTA streams one contiguous range and flushes
// its shared table at every tree (frame group) boundary inside it.
//  * candidate A: the range split evenly over the resident CTAs (at least
//    4 units per thread, but never more than one tree when trees are
//    smaller than that -- a tiny-frame CTA would otherwise flush 3-4 times);
//  * candidate B (n_trees <= resident CTAs): every tree cut into k equal
//    chunks, so no CTA straddles a boundary (one flush each).
// Cost model per CTA: its units + ~1800 units of streaming time per flush
// (a flush is ~2 us; one SM streams ~900 units/us).  C1 (30 x 640x480, L5)
// takes B (141 CTAs with up to two flushes -> 120 with one); C2 / C3 keep A.
static int64_t choose_units_per_cta(int64_t total_units, int64_t upt, int64_t n_trees, int64_t max_ctas,
                                    int threads) {
  constexpr int64_t FLUSH_UNITS = 1800;
  int64_t a = (total_units + max_ctas - 1) / max_ctas;
  const int64_t amin = std::min(int64_t(threads) * 4, upt);
  if (a < amin) a = amin;
  const int64_t a_segs = std::min<int64_t>(n_trees, (a + upt - 1) / upt + 1);
  const int64_t cost_a = a + a_segs * FLUSH_UNITS;
  if (OBG_ALIGN_TREES && n_trees <= max_ctas) {
    const int64_t k = max_ctas / n_trees;
    const int64_t b = (upt + k - 1) / k;
    if (b >= std::min(int64_t(threads), upt) && b + FLUSH_UNITS < cost_a) return b;
  }
  return a;
}

template <int L>
static int launch_build_flat(const uint8_t* frames, int64_t units_per_frame, int64_t total_units, int group_size,
                             uint32_t* ws, uint32_t* out_pyr, int64_t n_trees, uint32_t* zero_cube, int64_t zero_words,
                             uint32_t* counts, cudaStream_t st, int levels_out) {
  constexpr bool SMEM = L <= 6;
  const size_t smem = SMEM ? size_t(Smem<L>::alloc_words) * 4 : 0;
  // one-time per instantiation: opt in to > 48 KB dynamic smem, cache occupancy
  static DevCache occ[2];
  int& blocks_per_sm = occ[counts ? 1 : 0]();
  if (blocks_per_sm == 0) {
    if (counts) {
      auto k = k_build_flat<L, SMEM, true>;
      CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      blocks_per_sm = occupancy(k, BUILD_BLOCK, smem);
    } else {
      auto k = k_build_flat<L, SMEM, false>;
      CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      blocks_per_sm = occupancy(k, BUILD_BLOCK, smem);
    }
  }
  const int64_t max_ctas = int64_t(sm_count()) * blocks_per_sm;
  // at least 4 units per thread per CTA so that tiny inputs use few CTAs
  const int64_t per_cta = choose_units_per_cta(total_units, units_per_frame * group_size, total_units / (units_per_frame * group_size), max_ctas, BUILD_BLOCK);
  if (per_cta >= (int64_t(1) << 31) - 2 * BUILD_BLOCK)
    return set_err(OBG_EUNSUPPORTED, "too many pixels per launch (%lld units per CTA)", (long long)per_cta);
  const int grid = int((total_units + per_cta - 1) / per_cta);
#if OBG_BUILD_RING
  if constexpr (SMEM) {
    if (!counts) {
      constexpr bool BYTES = OBG_BYTE_TABLE && L == 5;
      using P = RingPlan<L, BYTES, BUILD_BLOCK>;
      static DevCache attr;
      if (!attr()) {
        CUDA_TRY(cudaFuncSetAttribute(k_build_ring<L, BYTES>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(P::TOTAL)));
        attr() = 1;
      }
      k_build_ring<L, BYTES><<<grid, BUILD_BLOCK, P::TOTAL, st>>>(frames, units_per_frame, total_units, group_size,
                                                                  per_cta, ws, out_pyr, n_trees, zero_cube, zero_words,
                                                                  levels_out);
      LAUNCH_CHECK("k_build_ring");
      return OBG_OK;
    }
  }
#endif
#if OBG_BYTE_TABLE
  // L = 5 only: at L = 4 uniform-random frames lose more to bank conflicts
  // of the scattered byte stores than the lookups cost (A/B: L5 -2..-5 %,
  // L4 uniform +5 %)
  if constexpr (L == 5) {
    if (!counts) {
      const size_t smem_b = ByteTab<L>::BITS_OFF + size_t(Smem<L>::alloc_words) * 4;
      static DevCache attr;
      if (!attr()) {
        CUDA_TRY(cudaFuncSetAttribute(k_build_bytes<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_b)));
        attr() = 1;
      }
      k_build_bytes<L><<<grid, BUILD_BLOCK, smem_b, st>>>(frames, units_per_frame, total_units, group_size, per_cta,
                                                          ws, out_pyr, n_trees, zero_cube, zero_words, levels_out);
      LAUNCH_CHECK("k_build_bytes");
      return OBG_OK;
    }
  }
#endif
  if (counts)
    k_build_flat<L, SMEM, true><<<grid, BUILD_BLOCK, smem, st>>>(frames, units_per_frame, total_units, group_size,
                                                                 per_cta, ws, out_pyr, n_trees, zero_cube, zero_words, counts, levels_out);
  else
    k_build_flat<L, SMEM, false><<<grid, BUILD_BLOCK, smem, st>>>(frames, units_per_frame, total_units, group_size,
                                                                  per_cta, ws, out_pyr, n_trees, zero_cube, zero_words, nullptr, levels_out);
  LAUNCH_CHECK("k_build_flat");
  return OBG_OK;
}

// ---------------------------------------------------------------------------
// a13: per-leaf pixel occupancy counts (the optional out_counts of
// obg_build_presence, the restatement np.bincount of
// pack_codes per frame tree, reference model.py:107 / tests/test_model.py:22-26).
// A separate streaming pass, so counts never slow the presence build.  The
// CTA streams a contiguous unit range (tree segments as K1):
//   L <= 5: one shared atomicAdd per pixel into a histogram privatised per CTA
//           (8^L u32, cube order, 128 KB at L = 5), flushed to the tree's
//           path-order counts in HBM (global atomics, non-zero bins only) at
//           each segment end.  The shared atomic unit merges a warp's equal
//           addresses itself; __match_any_sync aggregation (OBG_HIST_AGG=1)
//           measured ~5x slower on mixed warps;
//   L >= 6: straight into the tree's counts in global memory (1 MB at L = 6,
//           8 MB at L = 7), run-length merged per thread and warp-reduced when
//           a whole warp adds to one bin (a single-colour hot spot).  Two
//           privatised L = 6 forms were built and measured slower
//           (profiles/ab_r02/r02_ab_hist6.txt): a histogram spread over the
//           distributed shared memory of an 8-CTA cluster (2.2-2.7x: remote
//           red.shared::cluster adds run at ~0.5 per SM-clock), and 8 bin
//           slices per unit range (equal on mixed frames, 2.7x on a
//           single-colour frame, whose adds all land in one slice's CTA).
// ---------------------------------------------------------------------------
constexpr int HIST_BLOCK = 1024;
#ifndef OBG_HIST_AGG
#define OBG_HIST_AGG 0            // 1: __match_any_sync aggregation everywhere (measured, slower)
#endif

// add `cnt` at bin `key` (all lanes call it together; `go` = lane has an add):
// shared memory -- plain atomics (the shared atomic unit merges equal
// addresses of a warp itself); global -- one warp-reduced add when every
// lane adds to the same bin (a single-colour hot spot), else per lane
template <bool SMEM>
__device__ __forceinline__ void hist_add(uint32_t* at, uint32_t key, uint32_t cnt, bool go, int lane) {
  if constexpr (SMEM) {
    if (go) atomicAdd(at, cnt);
  } else {
    const uint32_t k0 = __shfl_sync(0xFFFFFFFFu, key, 0);
    if (__all_sync(0xFFFFFFFFu, go && key == k0)) {
      const uint32_t sum = __reduce_add_sync(0xFFFFFFFFu, cnt);
      if (lane == 0) atomicAdd(at, sum);
    } else if (go) {
      atomicAdd(at, cnt);
    }
  }
}

template <int L, bool SMEM>
__device__ __forceinline__ void hist_unit(const uint32_t (&w)[12], bool valid, uint32_t* dst, int lane) {
#if OBG_HIST_AGG == 1
  // __match_any_sync warp aggregation of equal bins (the lowest peer adds the
  // peer count).  Measured and NOT the default: MATCH.ANY per pixel costs ~5x
  // on mixed warps (C4 uniform L5: 2.05 ms vs 0.35 ms for presence + counts)
  // and the shared atomic unit already merges a warp's equal addresses.
  for16([&](auto jc) {
    constexpr int j = decltype(jc)::value;
    const uint32_t idx = cube_idx<L>(pixel_word<j>(w));
    const uint32_t key = valid ? idx : 0xFFFFFFFFu;
    const uint32_t peers = __match_any_sync(0xFFFFFFFFu, key);
    if (valid && lane == __ffs(peers) - 1) atomicAdd(dst + (SMEM ? idx : cube_to_code(idx, L)), uint32_t(__popc(peers)));
  });
#else
  if constexpr (SMEM) {
    // privatised shared histogram: one plain shared atomic per pixel (A/B,
    // tools/ab.py: fastest on every scene incl. the single-colour hot spot)
    for16([&](auto jc) {
      constexpr int j = decltype(jc)::value;
      if (valid) atomicAdd(dst + cube_idx<L>(pixel_word<j>(w)), 1u);
    });
  } else {
    // global counts: run-length over the thread's 16 consecutive pixels (one
    // add per run of equal bins), and one warp-reduced add when all lanes
    // add to the same bin -- a single-colour frame would otherwise serialise
    // 32 same-address global atomics per instruction (C4 constant L6:
    // 10.4 ms -> 0.54 ms)
    uint32_t prev = 0, run = 0;
    for16([&](auto jc) {
      constexpr int j = decltype(jc)::value;
      const uint32_t pos = cube_to_code(cube_idx<L>(pixel_word<j>(w)), L);
      if constexpr (j == 0) {
        prev = pos;
        run = 1;
      } else {
        const bool change = pos != prev;
        hist_add<SMEM>(dst + prev, prev, run, valid && change, lane);
        run = change ? 1u : run + 1u;
        prev = pos;
      }
    });
    hist_add<SMEM>(dst + prev, prev, run, valid, lane);
  }
#endif
}

template <int L, bool SMEM>
__global__ void __launch_bounds__(HIST_BLOCK, 1)
k_hist(const uint8_t* __restrict__ frames, int64_t units_per_frame, int64_t total_units, int group_size,
       int64_t units_per_cta, uint32_t* __restrict__ counts) {
  extern __shared__ __align__(16) uint32_t s_hist[];
  constexpr uint32_t NB = 1u << (3 * L);
  const int64_t u_begin = int64_t(blockIdx.x) * units_per_cta;
  const int64_t u_end = min(total_units, u_begin + units_per_cta);
  if (u_begin >= u_end) return;
  if constexpr (SMEM) {
    for (uint32_t i = threadIdx.x; i < NB; i += HIST_BLOCK) s_hist[i] = 0u;
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int64_t upt = units_per_frame * group_size;
  int64_t u = u_begin;
  while (u < u_end) {
    const int64_t tree = u / upt;
    const int64_t seg_end = min(u_end, (tree + 1) * upt);
    uint32_t* dst = counts + tree * int64_t(NB);
    const int64_t seg_len = seg_end - u;
    const int32_t rel0 = int32_t(threadIdx.x) - lane;
    const int32_t n_it = seg_len > rel0 ? int32_t((seg_len - rel0 + HIST_BLOCK - 1) / HIST_BLOCK) : 0;
    const int32_t n_lane = seg_len > rel0 + lane ? int32_t((seg_len - rel0 - lane + HIST_BLOCK - 1) / HIST_BLOCK) : 0;
    constexpr int64_t STEP = 48 * int64_t(HIST_BLOCK);
    const uint8_t* fp = frames + 48 * (u + rel0 + lane);
    uint32_t* hdst = SMEM ? s_hist : dst;
    uint32_t wa[12], wb[12];
    if (0 < n_lane) load_unit_at(fp, wa);
    for (int32_t k = 0; k < n_it;) {
      if (k + 1 < n_lane) load_unit_at(fp + STEP, wb);
      hist_unit<L, SMEM>(wa, k < n_lane, hdst, lane);
      fp += STEP;
      if (++k >= n_it) break;
      if (k + 1 < n_lane) load_unit_at(fp + STEP, wa);
      hist_unit<L, SMEM>(wb, k < n_lane, hdst, lane);
      fp += STEP;
      ++k;
    }
    if constexpr (SMEM) {
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < NB; i += HIST_BLOCK) {
        const uint32_t c = s_hist[i];
        if (c) {
          atomicAdd(dst + cube_to_code(i, L), c);
          s_hist[i] = 0u;
        }
      }
      __syncthreads();
    }
    u = seg_end;
  }
}

// ---------------------------------------------------------------------------
// a13 at L = 6: a per-CTA HASHED shared-memory histogram.  8^6 u32 bins are
// 1 MB, four times shared memory, but a CTA's range of a natural scene touches
// only a few thousand leaves (C3: ~4 k of 262 144 per CTA segment), so the
// private histogram is an open-addressing table of 2^14 (key, count) slots
// (128 KB): a pixel run looks its leaf up (linear probing from a
// multiplicative hash, at most HH_PROBES slots), claims an empty slot with one
// atomicCAS the first time, and adds with one shared atomic.  What does not
// fit goes straight to the tree's counts in global memory, exactly as the
// unhashed path does (the total is the same whichever way an add goes); when a
// segment has sent HH_GIVE_UP adds that way (uniform-random frames fill the
// table in the first 1 % of a segment) the CTA stops probing for the rest of
// the segment.  At a segment end the table is flushed to the path-order counts
// and cleared.  A thread's 16 consecutive pixels are run-length merged first,
// and a warp whose lanes all add to one leaf (single-colour frames) reduces
// to one add, as in the global path.
// ---------------------------------------------------------------------------
#ifndef OBG_HIST_HASH
#define OBG_HIST_HASH 1
#endif
#ifdef OBG_HH_BUCKETS
#define OBG_HH_BUCKETS_DEFAULT OBG_HH_BUCKETS
#else
#define OBG_HH_BUCKETS_DEFAULT 1
#endif
constexpr uint32_t HH_LOG = 14, HH_SLOTS = 1u << HH_LOG, HH_EMPTY = 0xFFFFFFFFu;
constexpr int HH_PROBES = 6;
constexpr uint32_t HH_GIVE_UP = OBG_HH_BUCKETS_DEFAULT ? 32768 : 4096;   // full buckets spill a steady trickle (Poisson tail)

// One add of `cnt` to leaf `idx` (cube order); returns false if the table had
// no room.  The table is 2^12 buckets of four (key, count) slots: a lookup is
// ONE 16-byte read of the bucket's keys and four compares, so a warp does not
// iterate to the longest probe sequence of its 32 lanes (linear probing over
// single slots cost ~2.7 rounds per pixel run at a 25 % load factor: 50 warp
// instructions per pixel slot, profiles/r02_ncu_hist6_c3.md).  A new key takes
// the first empty slot of its bucket (atomicCAS, slots in order, so a key
// never lands twice); a full bucket sends the add to global memory.
#ifndef OBG_HH_BUCKETS
#define OBG_HH_BUCKETS 1
#endif
__device__ __forceinline__ bool hh_add(uint32_t* keys, uint32_t* cnts, uint32_t idx, uint32_t cnt) {
#if OBG_HH_BUCKETS
  const uint32_t b4 = ((idx * 0x9E3779B1u) >> (32 - (HH_LOG - 2))) * 4u;
  const uint4 k = *reinterpret_cast<const uint4*>(keys + b4);
  int slot = k.x == idx ? 0 : k.y == idx ? 1 : k.z == idx ? 2 : k.w == idx ? 3 : -1;
  if (slot < 0) {
#pragma unroll 1
    for (int t = 0; t < 4 && slot < 0; ++t) {
      uint32_t cur = *reinterpret_cast<volatile uint32_t*>(keys + b4 + t);
      if (cur == HH_EMPTY) {
        cur = atomicCAS(keys + b4 + t, HH_EMPTY, idx);               // the old key: EMPTY = claimed
        if (cur == HH_EMPTY) cur = idx;
      }
      if (cur == idx) slot = t;
    }
    if (slot < 0) return false;
  }
  atomicAdd(cnts + b4 + slot, cnt);
  return true;
#else
  uint32_t h = (idx * 0x9E3779B1u) >> (32 - HH_LOG);
#pragma unroll 1
  for (int p = 0; p < HH_PROBES; ++p) {
    uint32_t k = keys[h];
    if (k == HH_EMPTY) k = atomicCAS(keys + h, HH_EMPTY, idx);     // returns the old key: EMPTY = claimed
    if (k == idx || k == HH_EMPTY) {
      atomicAdd(cnts + h, cnt);
      return true;
    }
    h = (h + 1u) & (HH_SLOTS - 1u);
  }
  return false;
#endif
}

template <int L>
__global__ void __launch_bounds__(HIST_BLOCK, 1)
k_hist_hash(const uint8_t* __restrict__ frames, int64_t units_per_frame, int64_t total_units, int group_size,
            int64_t units_per_cta, uint32_t* __restrict__ counts) {
  extern __shared__ __align__(16) uint32_t s_hh[];
  uint32_t* keys = s_hh;
  uint32_t* cnts = s_hh + HH_SLOTS;
  uint32_t* s_spill = s_hh + 2 * HH_SLOTS;             // adds of this segment that went to global memory
  constexpr int64_t NB = int64_t(1) << (3 * L);
  const int64_t u_begin = int64_t(blockIdx.x) * units_per_cta;
  const int64_t u_end = min(total_units, u_begin + units_per_cta);
  if (u_begin >= u_end) return;
  for (uint32_t i = threadIdx.x; i < HH_SLOTS; i += HIST_BLOCK) {
    keys[i] = HH_EMPTY;
    cnts[i] = 0u;
  }
  if (threadIdx.x == 0) *s_spill = 0u;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t upt = units_per_frame * group_size;
  int64_t u = u_begin;
  while (u < u_end) {
    const int64_t tree = u / upt;
    const int64_t seg_end = min(u_end, (tree + 1) * upt);
    uint32_t* dst = counts + tree * NB;
    const int64_t seg_len = seg_end - u;
    const int32_t rel0 = int32_t(threadIdx.x) - lane;
    const int32_t n_it = seg_len > rel0 ? int32_t((seg_len - rel0 + HIST_BLOCK - 1) / HIST_BLOCK) : 0;
    const int32_t n_lane = seg_len > rel0 + lane ? int32_t((seg_len - rel0 - lane + HIST_BLOCK - 1) / HIST_BLOCK) : 0;
    constexpr int64_t STEP = 48 * int64_t(HIST_BLOCK);
    const uint8_t* fp = frames + 48 * (u + rel0 + lane);
    // one run of `run` pixels of leaf `idx` (`go` = this lane has one)
    auto add_run = [&](uint32_t idx, uint32_t run, bool go, bool hashed) {
      if (go) {
        if (!(hashed && hh_add(keys, cnts, idx, run))) {
          atomicAdd(dst + cube_to_code(idx, L), run);
          if (hashed) atomicAdd(s_spill, 1u);
        }
      }
    };
    auto unit = [&](const uint32_t (&w)[12], bool valid) {
      const bool hashed = *reinterpret_cast<volatile uint32_t*>(s_spill) < HH_GIVE_UP;
      uint32_t prev = 0, run = 0;
      for16([&](auto jc) {
        constexpr int j = decltype(jc)::value;
        const uint32_t idx = cube_idx<L>(pixel_word<j>(w));
        if constexpr (j == 0) {
          prev = idx;
          run = 1;
        } else {
          const bool change = idx != prev;
          add_run(prev, run, valid && change, hashed);
          run = change ? 1u : run + 1u;
          prev = idx;
        }
      });
      // the unit's last run; when every lane's whole unit is one run of one
      // leaf (single-colour frames) the warp reduces to a single add
      const uint32_t i0 = __shfl_sync(0xFFFFFFFFu, prev, 0);
      const bool one = __all_sync(0xFFFFFFFFu, valid && run == 16u && prev == i0);
      add_run(prev, one ? 16u * 32u : run, one ? lane == 0 : valid, hashed);
    };
    uint32_t wa[12], wb[12];
    if (0 < n_lane) load_unit_at(fp, wa);
    for (int32_t k = 0; k < n_it;) {
      if (k + 1 < n_lane) load_unit_at(fp + STEP, wb);
      unit(wa, k < n_lane);
      fp += STEP;
      if (++k >= n_it) break;
      if (k + 1 < n_lane) load_unit_at(fp + STEP, wa);
      unit(wb, k < n_lane);
      fp += STEP;
      ++k;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < HH_SLOTS; i += HIST_BLOCK) {
      const uint32_t k = keys[i];
      if (k != HH_EMPTY) {
        atomicAdd(dst + cube_to_code(k, L), cnts[i]);
        keys[i] = HH_EMPTY;
        cnts[i] = 0u;
      }
    }
    if (threadIdx.x == 0) *s_spill = 0u;
    __syncthreads();
    u = seg_end;
  }
}

// (A/B variant, OBG_HIST_CLUSTER=1; slower than the global atomics, see above)
// L = 6: the 8^6-bin u32 histogram (1 MB) is privatised per CLUSTER of 8 CTAs
// in distributed shared memory -- each CTA holds 1/8 of the bins (128 KB) and
// the cluster streams one unit range as 8192 threads; every pixel sends one
// red.shared::cluster.add to the CTA owning its bin.  Owner = (R' ^ G' ^ B') & 7
// (a smooth scene spreads over all eight), bin within the owner = cube idx >> 3
// (B' & 7 is recovered from the owner, so the map is a bijection).  A thread's
// 16 consecutive pixels are run-length merged first (one add per run), which
// keeps a single-colour frame from sending 16 adds per thread to one address.
// At a tree-segment end: cluster barrier (release/acquire: every add landed),
// each CTA flushes its non-zero bins to the tree's path-order counts in HBM,
// barrier again before the next segment's adds.
constexpr int HC_CLUSTER = 8;
constexpr int HC_THREADS = HC_CLUSTER * HIST_BLOCK;
#ifndef OBG_HIST_CLUSTER
#define OBG_HIST_CLUSTER 0        // L = 6: 0 global atomics, 1 cluster DSMEM, 2 bin slices (A/B: 0 wins)
#endif

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// add `cnt` to bin `idx` (cube order, L = 6) of the cluster's histogram
__device__ __forceinline__ void hc_add(uint32_t s_base, uint32_t idx, uint32_t cnt) {
  const uint32_t owner = (idx ^ (idx >> 6) ^ (idx >> 12)) & 7u;
  const uint32_t local = s_base + ((idx >> 3) << 2);
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(owner));
  asm volatile("red.shared::cluster.add.u32 [%0], %1;" :: "r"(remote), "r"(cnt) : "memory");
}

__device__ __forceinline__ void hc_unit(const uint32_t (&w)[12], bool valid, uint32_t s_base) {
  uint32_t prev = 0, run = 0;
  for16([&](auto jc) {
    constexpr int j = decltype(jc)::value;
    const uint32_t idx = cube_idx<6>(pixel_word<j>(w));
    if constexpr (j == 0) {
      prev = idx;
      run = 1;
    } else {
      const bool change = idx != prev;
      if (valid && change) hc_add(s_base, prev, run);
      run = change ? 1u : run + 1u;
      prev = idx;
    }
  });
  if (valid) hc_add(s_base, prev, run);
}

__global__ void __launch_bounds__(HIST_BLOCK, 1)
k_hist_cluster(const uint8_t* __restrict__ frames, int64_t units_per_frame, int64_t total_units, int group_size,
               int64_t units_per_cluster, uint32_t* __restrict__ counts) {
  extern __shared__ __align__(16) uint32_t s_hist[];
  constexpr int L = 6;
  constexpr uint32_t NB = 1u << (3 * L), NLOC = NB / HC_CLUSTER;
  const uint32_t rank = cluster_rank();
  const int64_t cl = int64_t(blockIdx.x) / HC_CLUSTER;
  const int64_t u_begin = cl * units_per_cluster;
  const int64_t u_end = min(total_units, u_begin + units_per_cluster);
  if (u_begin >= u_end) return;                  // uniform over the cluster
  for (uint32_t i = threadIdx.x; i < NLOC; i += HIST_BLOCK) s_hist[i] = 0u;
  const uint32_t s_base = uint32_t(__cvta_generic_to_shared(s_hist));
  cluster_sync_all();                            // every slice zeroed before the first add
  const int lane = threadIdx.x & 31;
  const int32_t gt = int32_t(rank) * HIST_BLOCK + int32_t(threadIdx.x);   // thread of the cluster
  const int64_t upt = units_per_frame * group_size;
  int64_t u = u_begin;
  while (u < u_end) {
    const int64_t tree = u / upt;
    const int64_t seg_end = min(u_end, (tree + 1) * upt);
    uint32_t* dst = counts + tree * int64_t(NB);
    const int64_t seg_len = seg_end - u;
    const int32_t rel0 = gt - lane;
    const int32_t n_it = seg_len > rel0 ? int32_t((seg_len - rel0 + HC_THREADS - 1) / HC_THREADS) : 0;
    const int32_t n_lane = seg_len > rel0 + lane ? int32_t((seg_len - rel0 - lane + HC_THREADS - 1) / HC_THREADS) : 0;
    constexpr int64_t STEP = 48 * int64_t(HC_THREADS);
    const uint8_t* fp = frames + 48 * (u + rel0 + lane);
    uint32_t wa[12], wb[12];
    if (0 < n_lane) load_unit_at(fp, wa);
    for (int32_t k = 0; k < n_it;) {
      if (k + 1 < n_lane) load_unit_at(fp + STEP, wb);
      hc_unit(wa, k < n_lane, s_base);
      fp += STEP;
      if (++k >= n_it) break;
      if (k + 1 < n_lane) load_unit_at(fp + STEP, wa);
      hc_unit(wb, k < n_lane, s_base);
      fp += STEP;
      ++k;
    }
    cluster_sync_all();                          // all adds of the segment landed
    for (uint32_t i = threadIdx.x; i < NLOC; i += HIST_BLOCK) {
      const uint32_t c = s_hist[i];
      if (c) {
        const uint32_t rg = i >> 3;              // R' << 6 | G'
        const uint32_t b = ((i & 7u) << 3) | ((rank ^ rg ^ (rg >> 6)) & 7u);
        atomicAdd(dst + cube_to_code((rg << 6) | b, L), c);
        s_hist[i] = 0u;
      }
    }
    cluster_sync_all();                          // slices clear before the next segment's adds
    u = seg_end;
  }
}

static int launch_hist_cluster(const uint8_t* frames, int64_t units_per_frame, int64_t total_units, int group_size,
                               uint32_t* counts, cudaStream_t st) {
  constexpr size_t smem = (size_t(1) << 18) / HC_CLUSTER * 4;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = HC_CLUSTER;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(HIST_BLOCK);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  static DevCache max_clusters;
  if (!max_clusters()) {
    CUDA_TRY(cudaFuncSetAttribute(k_hist_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    cfg.gridDim = dim3(HC_CLUSTER * 64);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k_hist_cluster, &cfg) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 1;
    }
    max_clusters() = n;
  }
  const int64_t upt = units_per_frame * group_size;
  const int64_t per_cl = choose_units_per_cta(total_units, upt, total_units / upt, max_clusters(), HC_THREADS);
  if (per_cl >= (int64_t(1) << 31) - 2 * HC_THREADS)
    return set_err(OBG_EUNSUPPORTED, "too many pixels per launch (%lld units per cluster)", (long long)per_cl);
  const int n_cl = int((total_units + per_cl - 1) / per_cl);
  cfg.gridDim = dim3(unsigned(n_cl * HC_CLUSTER));
  CUDA_TRY(cudaLaunchKernelEx(&cfg, k_hist_cluster, frames, units_per_frame, total_units, group_size, per_cl, counts));
  LAUNCH_CHECK("k_hist_cluster");
  return OBG_OK;
}

// (A/B variant, OBG_HIST_CLUSTER=2; slower than the global atomics, see above)
// L = 6, bin slices: 8 CTAs share one unit range (adjacent blockIdx, so they
// run in the same wave and 7 of the 8 frame reads hit L2); CTA s privatises
// the bins with B' & 7 == s (128 KB, bin = idx >> 3) and streams the whole
// range, one local shared atomic per pixel of its slice.
__global__ void __launch_bounds__(HIST_BLOCK, 1)
k_hist_slices(const uint8_t* __restrict__ frames, int64_t units_per_frame, int64_t total_units, int group_size,
              int64_t units_per_range, uint32_t* __restrict__ counts) {
  extern __shared__ __align__(16) uint32_t s_hist[];
  constexpr int L = 6;
  constexpr uint32_t NB = 1u << (3 * L), NLOC = NB / HC_CLUSTER;
  const uint32_t slice = blockIdx.x % HC_CLUSTER;
  const int64_t u_begin = int64_t(blockIdx.x / HC_CLUSTER) * units_per_range;
  const int64_t u_end = min(total_units, u_begin + units_per_range);
  if (u_begin >= u_end) return;
  for (uint32_t i = threadIdx.x; i < NLOC; i += HIST_BLOCK) s_hist[i] = 0u;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t upt = units_per_frame * group_size;
  int64_t u = u_begin;
  while (u < u_end) {
    const int64_t tree = u / upt;
    const int64_t seg_end = min(u_end, (tree + 1) * upt);
    uint32_t* dst = counts + tree * int64_t(NB);
    const int64_t seg_len = seg_end - u;
    const int32_t rel0 = int32_t(threadIdx.x) - lane;
    const int32_t n_it = seg_len > rel0 ? int32_t((seg_len - rel0 + HIST_BLOCK - 1) / HIST_BLOCK) : 0;
    const int32_t n_lane = seg_len > rel0 + lane ? int32_t((seg_len - rel0 - lane + HIST_BLOCK - 1) / HIST_BLOCK) : 0;
    constexpr int64_t STEP = 48 * int64_t(HIST_BLOCK);
    const uint8_t* fp = frames + 48 * (u + rel0 + lane);
    uint32_t wa[12], wb[12];
    auto body = [&](const uint32_t (&w)[12], bool valid) {
      for16([&](auto jc) {
        constexpr int j = decltype(jc)::value;
        const uint32_t idx = cube_idx<L>(pixel_word<j>(w));
        if (valid && (idx & 7u) == slice) atomicAdd(s_hist + (idx >> 3), 1u);
      });
    };
    if (0 < n_lane) load_unit_at(fp, wa);
    for (int32_t k = 0; k < n_it;) {
      if (k + 1 < n_lane) load_unit_at(fp + STEP, wb);
      body(wa, k < n_lane);
      fp += STEP;
      if (++k >= n_it) break;
      if (k + 1 < n_lane) load_unit_at(fp + STEP, wa);
      body(wb, k < n_lane);
      fp += STEP;
      ++k;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < NLOC; i += HIST_BLOCK) {
      const uint32_t c = s_hist[i];
      if (c) {
        atomicAdd(dst + cube_to_code((i << 3) | slice, L), c);
        s_hist[i] = 0u;
      }
    }
    __syncthreads();
    u = seg_end;
  }
}

static int launch_hist_slices(const uint8_t* frames, int64_t units_per_frame, int64_t total_units, int group_size,
                              uint32_t* counts, cudaStream_t st) {
  constexpr size_t smem = (size_t(1) << 18) / HC_CLUSTER * 4;
  static DevCache attr;
  if (!attr()) {
    CUDA_TRY(cudaFuncSetAttribute(k_hist_slices, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr() = 1;
  }
  const int64_t n_ranges_max = std::max(1, sm_count() / HC_CLUSTER);
  const int64_t upt = units_per_frame * group_size;
  const int64_t per_r = choose_units_per_cta(total_units, upt, total_units / upt, n_ranges_max, HIST_BLOCK);
  if (per_r >= (int64_t(1) << 31) - 2 * HIST_BLOCK)
    return set_err(OBG_EUNSUPPORTED, "too many pixels per launch (%lld units per range)", (long long)per_r);
  const int n_r = int((total_units + per_r - 1) / per_r);
  k_hist_slices<<<n_r * HC_CLUSTER, HIST_BLOCK, smem, st>>>(frames, units_per_frame, total_units, group_size, per_r,
                                                           counts);
  LAUNCH_CHECK("k_hist_slices");
  return OBG_OK;
}

template <int L>
static int launch_hist(const uint8_t* frames, int64_t units_per_frame, int64_t total_units, int group_size,
                       uint32_t* counts, cudaStream_t st) {
  if constexpr (L == 6) {
    if (OBG_HIST_CLUSTER == 1) return launch_hist_cluster(frames, units_per_frame, total_units, group_size, counts, st);
    if (OBG_HIST_CLUSTER == 2) return launch_hist_slices(frames, units_per_frame, total_units, group_size, counts, st);
  }
  constexpr bool SMEM = L <= 5;
  if constexpr (L == 6 && OBG_HIST_HASH) {      // L >= 7: a CTA segment of a natural scene overflows the table (A/B: C3 scene at L7 +50 %)
    constexpr size_t smem_h = (2 * size_t(HH_SLOTS) + 4) * 4;
    static DevCache attr_h;
    if (!attr_h()) {
      CUDA_TRY(cudaFuncSetAttribute(k_hist_hash<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_h)));
      attr_h() = 1;
    }
    const int64_t upt = units_per_frame * group_size;
    const int64_t per_h = choose_units_per_cta(total_units, upt, total_units / upt, sm_count(), HIST_BLOCK);
    if (per_h >= (int64_t(1) << 31) - 2 * HIST_BLOCK)
      return set_err(OBG_EUNSUPPORTED, "too many pixels per launch (%lld units per CTA)", (long long)per_h);
    k_hist_hash<L><<<int((total_units + per_h - 1) / per_h), HIST_BLOCK, smem_h, st>>>(frames, units_per_frame,
                                                                                      total_units, group_size, per_h,
                                                                                      counts);
    LAUNCH_CHECK("k_hist_hash");
    return OBG_OK;
  }
  const size_t smem = SMEM ? (size_t(1) << (3 * L)) * 4 : 0;
  static DevCache attr;
  if (!attr()) {
    if (smem > 48 * 1024)
      CUDA_TRY(cudaFuncSetAttribute(k_hist<L, SMEM>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr() = occupancy(k_hist<L, SMEM>, HIST_BLOCK, smem);
  }
  const int64_t max_ctas = int64_t(sm_count()) * attr();
  const int64_t per_cta = choose_units_per_cta(total_units, units_per_frame * group_size, total_units / (units_per_frame * group_size), max_ctas, HIST_BLOCK);
  if (per_cta >= (int64_t(1) << 31) - 2 * HIST_BLOCK)
    return set_err(OBG_EUNSUPPORTED, "too many pixels per launch (%lld units per CTA)", (long long)per_cta);
  const int grid = int((total_units + per_cta - 1) / per_cta);
  k_hist<L, SMEM><<<grid, HIST_BLOCK, smem, st>>>(frames, units_per_frame, total_units, group_size, per_cta, counts);
  LAUNCH_CHECK("k_hist");
  return OBG_OK;
}

static int launch_hist_any(int L, const uint8_t* frames, int64_t upf, int64_t total_units, int group_size,
                           uint32_t* counts, cudaStream_t st) {
  switch (L) {
    case 1: return launch_hist<1>(frames, upf, total_units, group_size, counts, st);
    case 2: return launch_hist<2>(frames, upf, total_units, group_size, counts, st);
    case 3: return launch_hist<3>(frames, upf, total_units, group_size, counts, st);
    case 4: return launch_hist<4>(frames, upf, total_units, group_size, counts, st);
    case 5: return launch_hist<5>(frames, upf, total_units, group_size, counts, st);
    case 6: return launch_hist<6>(frames, upf, total_units, group_size, counts, st);
    case 7: return launch_hist<7>(frames, upf, total_units, group_size, counts, st);
    default: return launch_hist<8>(frames, upf, total_units, group_size, counts, st);
  }
}

#ifndef OBG_L7_ONEPASS
#define OBG_L7_ONEPASS 1
#endif
static int launch_build_l7h(const uint8_t* frames, int64_t units_per_frame, int64_t total_units, int group_size,
                            uint32_t* ws, uint32_t* out_pyr, int64_t n_trees, uint32_t* zero_cube, int64_t zero_words,
                            cudaStream_t st) {
  if (OBG_L7_ONEPASS) {
    constexpr size_t smem = size_t(L7C_WORDS) * 4;
    static DevCache attr;
    if (!attr()) {
      CUDA_TRY(cudaFuncSetAttribute(k_build_l7c, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      attr() = 1;
    }
    const int64_t max_ctas = sm_count();
    const int64_t per_cta = choose_units_per_cta(total_units, units_per_frame * group_size,
                                                 total_units / (units_per_frame * group_size), max_ctas, L7C_BLOCK);
    if (per_cta >= (int64_t(1) << 31) - 2 * L7C_BLOCK)
      return set_err(OBG_EUNSUPPORTED, "too many pixels per launch (%lld units per CTA)", (long long)per_cta);
    const int grid = int((total_units + per_cta - 1) / per_cta);
    k_build_l7c<<<grid, L7C_BLOCK, smem, st>>>(frames, units_per_frame, total_units, group_size, per_cta, ws, out_pyr,
                                               n_trees, zero_cube, zero_words);
    LAUNCH_CHECK("k_build_l7c");
    return OBG_OK;
  }
  constexpr size_t smem = size_t(L7H_ALLOC) * 4;
  static DevCache attr;
  if (!attr()) {
    CUDA_TRY(cudaFuncSetAttribute(k_build_l7h, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr() = 1;
  }
  const int64_t max_ctas = sm_count();                   // one CTA per SM
  const int64_t per_cta = choose_units_per_cta(total_units, units_per_frame * group_size, total_units / (units_per_frame * group_size), max_ctas, L7H_BLOCK);
  if (per_cta >= (int64_t(1) << 31) - 2 * L7H_BLOCK)
    return set_err(OBG_EUNSUPPORTED, "too many pixels per launch (%lld units per CTA)", (long long)per_cta);
  const int grid = int((total_units + per_cta - 1) / per_cta);
  k_build_l7h<<<grid, L7H_BLOCK, smem, st>>>(frames, units_per_frame, total_units, group_size, per_cta, ws, out_pyr,
                                             n_trees, zero_cube, zero_words);
  LAUNCH_CHECK("k_build_l7h");
  return OBG_OK;
}

static int launch_pyramid(const uint32_t* src, int64_t src_stride, bool from_cube, int64_t n_trees, int L,
                          uint32_t* out, cudaStream_t st) {
  const int64_t LW = level_words(L);
  const int64_t nw = LW < PYR_CHUNK ? LW : PYR_CHUNK;
  dim3 grid(unsigned(LW / nw), unsigned(n_trees));
  if (n_trees > 65535) return set_err(OBG_EUNSUPPORTED, "too many trees in one call (%lld > 65535)", (long long)n_trees);
  if (from_cube) k_pyramid<true><<<grid, PYR_BLOCK, 0, st>>>(src, src_stride, L, out);
  else k_pyramid<false><<<grid, PYR_BLOCK, 0, st>>>(src, src_stride, L, out);
  LAUNCH_CHECK("k_pyramid");
  return OBG_OK;
}

static int merge_common(const uint32_t* pyramids, int n_trees, int n_regions, int levels, int64_t k_min,
                        uint32_t* counts, uint32_t* out, uint32_t* out_cube, int flags, void* stream);
static int finish_operand(uint32_t* operand, int64_t n_regions, int levels, cudaStream_t st);

// cube_levels: obg_build_model's flow -- K1, then k_levels_cube (cube-order
// levels below the leaves into out_pyramids; leaves stay in the workspace)
// instead of k_pyramid.
static int build_presence_impl(const uint8_t* frames, int n_frames, int height, int width, int levels, int grid_rows,
                               int grid_cols, int group_size, uint32_t* out_pyramids, uint32_t* out_counts,
                               void* workspace, int64_t workspace_bytes, int flags, uint32_t* zero_cube,
                               int64_t zero_words, void* stream, bool cube_levels = false) {
  if (levels < 1 || levels > 8) return set_err(OBG_EINVAL, "levels must be in 1..8, got %d", levels);
  if (n_frames < 1) return set_err(OBG_EINVAL, "no frames given");
  if (height < 1 || width < 1) return set_err(OBG_EINVAL, "frame dimensions must be >= 1");
  if (grid_rows < 1 || grid_cols < 1) return set_err(OBG_EINVAL, "grid dimensions must be >= 1");
  if (group_size < 1) return set_err(OBG_EINVAL, "group_size must be >= 1");
  const int n_groups = n_frames / group_size;
  if (n_groups == 0)
    return set_err(OBG_EINVAL, "need at least %d frames for one group, got %d", group_size, n_frames);
  if (!frames || !out_pyramids || !workspace) return set_err(OBG_EINVAL, "null buffer");
  const int64_t n_regions = int64_t(grid_rows) * grid_cols;
  const int64_t n_trees = int64_t(n_groups) * n_regions;
  const int64_t need = obg_build_workspace_bytes(n_groups, int(n_regions), levels);
  if (workspace_bytes < need)
    return set_err(OBG_EINVAL, "workspace too small: %lld < %lld bytes", (long long)workspace_bytes, (long long)need);
  cudaStream_t st = as_stream(stream);
  uint32_t* ws = static_cast<uint32_t*>(workspace);
  const int64_t CW = cube_words(levels);
  const int64_t PW = pyr_words(levels);
  const int64_t P = int64_t(height) * width;
  const int64_t used_pixels = int64_t(n_groups) * group_size * P;
  const bool flat = n_regions == 1 && (P % 16) == 0 && (reinterpret_cast<uintptr_t>(frames) % 16) == 0;
  // trees whose leading pyramid words K1 clears for k_pyramid's atomics
  const int64_t clear_trees = cube_levels ? 0 : n_trees;
  // flat L <= 6: K1 writes the cube-order upper levels itself (k_build_flat flush)
  const bool band = !flat && n_regions > 1 && levels <= 6 && !out_counts && (width % 16) == 0 &&
                    (reinterpret_cast<uintptr_t>(frames) % 16) == 0 && grid_cols <= 16 &&
                    int64_t(grid_cols) * 4 * (levels == 6 ? BandBits<6>::ALLOC : BandBits<5>::ALLOC) + 68 <= 227 * 1024;
  const int smem_levels = (cube_levels && (flat || band) && levels <= 6) ? 1 : 0;
  // The workspace is handed back all-zero by k_pyramid; a caller that keeps
  // it (OBG_WS_ZEROED) skips the clear.  Output pyramids need no memset: every
  // word is either stored once or (leading shared words) cleared by K1.
  if (!(flags & OBG_WS_ZEROED)) CUDA_TRY(cudaMemsetAsync(ws, 0, size_t(n_trees * ws_words(levels) * 4), st));
  if (out_counts) CUDA_TRY(cudaMemsetAsync(out_counts, 0, size_t(n_trees) * (size_t(1) << (3 * levels)) * 4, st));
  int rc = OBG_OK;
  if (flat && out_counts) {
    // presence through the fast kernels, counts in their own streaming pass
    const int64_t upf = P / 16, total_units = used_pixels / 16;
    rc = launch_hist_any(levels, frames, upf, total_units, group_size, out_counts, st);
    if (rc != OBG_OK) return rc;
    out_counts = nullptr;
  }
  if (flat) {
    const int64_t upf = P / 16, total_units = used_pixels / 16;
    switch (levels) {
      case 1: rc = launch_build_flat<1>(frames, upf, total_units, group_size, ws, out_pyramids, clear_trees, zero_cube, zero_words, out_counts, st, smem_levels); break;
      case 2: rc = launch_build_flat<2>(frames, upf, total_units, group_size, ws, out_pyramids, clear_trees, zero_cube, zero_words, out_counts, st, smem_levels); break;
      case 3: rc = launch_build_flat<3>(frames, upf, total_units, group_size, ws, out_pyramids, clear_trees, zero_cube, zero_words, out_counts, st, smem_levels); break;
      case 4: rc = launch_build_flat<4>(frames, upf, total_units, group_size, ws, out_pyramids, clear_trees, zero_cube, zero_words, out_counts, st, smem_levels); break;
      case 5: rc = launch_build_flat<5>(frames, upf, total_units, group_size, ws, out_pyramids, clear_trees, zero_cube, zero_words, out_counts, st, smem_levels); break;
      case 6: rc = launch_build_flat<6>(frames, upf, total_units, group_size, ws, out_pyramids, clear_trees, zero_cube, zero_words, out_counts, st, smem_levels); break;
      case 7:
        rc = out_counts ? launch_build_flat<7>(frames, upf, total_units, group_size, ws, out_pyramids, clear_trees,
                                               zero_cube, zero_words, out_counts, st, smem_levels)
                        : launch_build_l7h(frames, upf, total_units, group_size, ws, out_pyramids, clear_trees,
                                           zero_cube, zero_words, st);
        break;
      default: rc = launch_build_flat<8>(frames, upf, total_units, group_size, ws, out_pyramids, clear_trees, zero_cube, zero_words, out_counts, st, smem_levels); break;
    }
  } else if (band) {
    const int nf = n_groups * group_size;
    switch (levels) {
      case 1: rc = launch_build_band<1>(frames, nf, height, width, grid_rows, grid_cols, group_size, ws, out_pyramids, clear_trees, zero_cube, zero_words, st, smem_levels); break;
      case 2: rc = launch_build_band<2>(frames, nf, height, width, grid_rows, grid_cols, group_size, ws, out_pyramids, clear_trees, zero_cube, zero_words, st, smem_levels); break;
      case 3: rc = launch_build_band<3>(frames, nf, height, width, grid_rows, grid_cols, group_size, ws, out_pyramids, clear_trees, zero_cube, zero_words, st, smem_levels); break;
      case 4: rc = launch_build_band<4>(frames, nf, height, width, grid_rows, grid_cols, group_size, ws, out_pyramids, clear_trees, zero_cube, zero_words, st, smem_levels); break;
      case 5: rc = launch_build_band<5>(frames, nf, height, width, grid_rows, grid_cols, group_size, ws, out_pyramids, clear_trees, zero_cube, zero_words, st, smem_levels); break;
      default: rc = launch_build_band<6>(frames, nf, height, width, grid_rows, grid_cols, group_size, ws, out_pyramids, clear_trees, zero_cube, zero_words, st, smem_levels); break;
    }
  } else {
    const int grid = grid_for(used_pixels, 256, sm_count() * 8);
    if (out_counts)
      k_build_generic<true><<<grid, 256, 0, st>>>(frames, used_pixels, height, width, levels, grid_rows, grid_cols,
                                                   group_size, ws, out_pyramids, clear_trees, zero_cube, zero_words, out_counts);
    else
      k_build_generic<false><<<grid, 256, 0, st>>>(frames, used_pixels, height, width, levels, grid_rows, grid_cols,
                                                    group_size, ws, out_pyramids, clear_trees, zero_cube, zero_words, nullptr);
    LAUNCH_CHECK("k_build_generic");
  }
  if (rc != OBG_OK) return rc;
  if (cube_levels) {
    if (levels > 1 && !smem_levels) {
      k_levels_cube<<<unsigned(n_trees), LVL_BLOCK, 0, st>>>(ws, levels);
      LAUNCH_CHECK("k_levels_cube");
    }
    return OBG_OK;
  }
  return launch_pyramid(ws, ws_words(levels), true, n_trees, levels, out_pyramids, st);
}

int obg_build_presence(const uint8_t* frames, int n_frames, int height, int width, int levels, int grid_rows,
                       int grid_cols, int group_size, uint32_t* out_pyramids, uint32_t* out_counts, void* workspace,
                       int64_t workspace_bytes, int flags, void* stream) {
  g_err[0] = 0;
  return build_presence_impl(frames, n_frames, height, width, levels, grid_rows, grid_cols, group_size, out_pyramids,
                             out_counts, workspace, workspace_bytes, flags, nullptr, 0, stream);
}

int obg_build_model(const uint8_t* frames, int n_frames, int height, int width, int levels, int grid_rows,
                    int grid_cols, int group_size, int64_t k_min, uint32_t* tree_pyramids, uint32_t* out_merged,
                    uint32_t* out_cube, void* workspace, int64_t workspace_bytes, int flags, void* stream) {
  g_err[0] = 0;
  if (k_min < 1) return set_err(OBG_EINVAL, "k_min must be >= 1, got %lld", (long long)k_min);
  if (!out_merged || !out_cube) return set_err(OBG_EINVAL, "null buffer");
  if (levels < 1 || levels > 8) return set_err(OBG_EINVAL, "levels must be in 1..8, got %d", levels);
  if (!tree_pyramids) return set_err(OBG_EINVAL, "null buffer");
  const int64_t n_regions = int64_t(grid_rows) * grid_cols;
  // K1 (+ cube-order levels), K3f (merge; stores every operand and merged
  // pyramid word and zeroes the workspace): no memsets at all
  int rc = build_presence_impl(frames, n_frames, height, width, levels, grid_rows, grid_cols, group_size,
                               tree_pyramids, nullptr, workspace, workspace_bytes, flags, nullptr, 0, stream,
                               /*cube_levels=*/true);
  if (rc != OBG_OK) return rc;
  cudaStream_t st = as_stream(stream);
  const int n_groups = n_frames / group_size;
  const int64_t words = pyr_words(levels) * n_regions;
  if (n_regions > 65535) return set_err(OBG_EUNSUPPORTED, "too many regions (%lld > 65535)", (long long)n_regions);
  if (OBG_MERGE_CSA && n_groups <= MC_MAX_TREES) {
    int64_t blocks = 1;                                   // block 0: levels 1..2
    for (int l = 3; l <= levels; ++l) blocks += (level_words(l) + MC_SLOTS - 1) / MC_SLOTS;
    // a programmatic dependent of the build kernel just launched on `st`
    cudaError_t le = launch_dep(k_merge_tiles, dim3(unsigned(blocks), unsigned(n_regions)), dim3(MC_BLOCK), 0, st, 1,
                                static_cast<uint32_t*>(workspace), n_groups, int(n_regions), levels, k_min, out_cube,
                                out_merged);
    if (le != cudaSuccess) return set_err(OBG_ECUDA, "launch of k_merge_tiles failed: %s", cudaGetErrorString(le));
    LAUNCH_CHECK("k_merge_tiles");
  } else {
    int64_t blocks = 1;                                   // block 0: levels 1..2
    for (int l = 3; l <= levels; ++l) blocks += mf_blocks(l);
    k_merge_fused<0><<<dim3(unsigned(blocks), unsigned(n_regions)), dim3(32, MERGE_GROUPS_C), 0, st>>>(
        static_cast<uint32_t*>(workspace), n_groups, int(n_regions), levels, k_min, out_cube, out_merged, nullptr);
    LAUNCH_CHECK("k_merge_fused");
  }
  (void)words;
  return finish_operand(out_cube, n_regions, levels, st);
}

int obg_pyramid_from_leaves(const uint32_t* leaves, int n_trees, int levels, uint32_t* out_pyramids, void* stream) {
  g_err[0] = 0;
  if (levels < 1 || levels > 8) return set_err(OBG_EINVAL, "levels must be in 1..8, got %d", levels);
  if (n_trees < 0) return set_err(OBG_EINVAL, "n_trees must be >= 0");
  if (n_trees == 0) return OBG_OK;
  if (!leaves || !out_pyramids) return set_err(OBG_EINVAL, "null buffer");
  cudaStream_t st = as_stream(stream);
  CUDA_TRY(cudaMemsetAsync(out_pyramids, 0, size_t(n_trees) * pyr_words(levels) * 4, st));
  return launch_pyramid(leaves, level_words(levels), false, n_trees, levels, out_pyramids, st);
}

int obg_prune(const uint32_t* pyramids, int n_trees, int levels, int new_levels, uint32_t* out_pyramids, void* stream) {
  g_err[0] = 0;
  if (levels < 1 || levels > 8) return set_err(OBG_EINVAL, "levels must be in 1..8, got %d", levels);
  if (new_levels < 1 || new_levels > levels)
    return set_err(OBG_EINVAL, "new_depth must be in 1..%d, got %d", levels, new_levels);
  if (n_trees < 0) return set_err(OBG_EINVAL, "n_trees must be >= 0");
  if (n_trees == 0) return OBG_OK;
  if (!pyramids || !out_pyramids) return set_err(OBG_EINVAL, "null buffer");
  const int64_t PW = pyr_words(levels), PW2 = pyr_words(new_levels);
  k_prune<<<grid_for(PW2 * n_trees, 256, sm_count() * 8), 256, 0, as_stream(stream)>>>(pyramids, PW, PW2, n_trees,
                                                                                       out_pyramids);
  LAUNCH_CHECK("k_prune");
  return OBG_OK;
}

static int finish_operand(uint32_t* operand, int64_t n_regions, int levels, cudaStream_t st) {
  if (levels != 7 || !operand) return OBG_OK;
  k_l7_states<<<unsigned(n_regions), 1024, 0, st>>>(operand);
  LAUNCH_CHECK("k_l7_states");
  return OBG_OK;
}

static int merge_common(const uint32_t* pyramids, int n_trees, int n_regions, int levels, int64_t k_min,
                        uint32_t* counts, uint32_t* out, uint32_t* out_cube, int flags, void* stream) {
  if (levels < 1 || levels > 8) return set_err(OBG_EINVAL, "levels must be in 1..8, got %d", levels);
  if (n_trees < 1) return set_err(OBG_EINVAL, "no trees to merge");
  if (n_regions < 1) return set_err(OBG_EINVAL, "n_regions must be >= 1");
  if (!pyramids) return set_err(OBG_EINVAL, "null buffer");
  cudaStream_t st = as_stream(stream);
  if (out_cube && !(flags & OBG_CUBE_ZEROED))
    CUDA_TRY(cudaMemsetAsync(out_cube, 0, size_t(n_regions) * operand_words(levels) * 4, st));
  const int64_t words = pyr_words(levels) * n_regions;
  k_merge<<<grid_for(words, 32, sm_count() * 16), dim3(32, MERGE_GROUPS), 0, st>>>(
      pyramids, n_trees, n_regions, levels, k_min, counts, out, out_cube);
  LAUNCH_CHECK("k_merge");
  return finish_operand(out_cube, n_regions, levels, st);
}

int obg_merge_counts(const uint32_t* pyramids, int n_trees, int n_regions, int levels, uint32_t* counts, void* stream) {
  g_err[0] = 0;
  if (!counts) return set_err(OBG_EINVAL, "null buffer");
  return merge_common(pyramids, n_trees, n_regions, levels, 0, counts, nullptr, nullptr, 0, stream);
}

int obg_merge(const uint32_t* pyramids, int n_trees, int n_regions, int levels, int64_t k_min,
              uint32_t* out_pyramids, uint32_t* out_cube, void* stream) {
  g_err[0] = 0;
  if (!out_pyramids) return set_err(OBG_EINVAL, "null buffer");
  if (k_min < 1) return set_err(OBG_EINVAL, "k_min must be >= 1, got %lld", (long long)k_min);
  return merge_common(pyramids, n_trees, n_regions, levels, k_min, nullptr, out_pyramids, out_cube, 0, stream);
}

int obg_merge_threshold(const uint32_t* counts, int n_regions, int levels, int64_t k_min, uint32_t* out_pyramids,
                        uint32_t* out_cube, void* stream) {
  g_err[0] = 0;
  if (levels < 1 || levels > 8) return set_err(OBG_EINVAL, "levels must be in 1..8, got %d", levels);
  if (n_regions < 1) return set_err(OBG_EINVAL, "n_regions must be >= 1");
  if (k_min < 1) return set_err(OBG_EINVAL, "k_min must be >= 1, got %lld", (long long)k_min);
  if (!counts || !out_pyramids) return set_err(OBG_EINVAL, "null buffer");
  cudaStream_t st = as_stream(stream);
  if (out_cube) CUDA_TRY(cudaMemsetAsync(out_cube, 0, size_t(n_regions) * operand_words(levels) * 4, st));
  const int64_t words = pyr_words(levels) * n_regions;
  k_threshold<<<grid_for(words, 256, sm_count() * 8), 256, 0, st>>>(counts, n_regions, levels, k_min,
                                                                   out_pyramids, out_cube);
  LAUNCH_CHECK("k_threshold");
  return finish_operand(out_cube, n_regions, levels, st);
}

int obg_leaf_cube(const uint32_t* pyramids, int n_trees, int levels, uint32_t* cube, void* stream) {
  g_err[0] = 0;
  if (levels < 1 || levels > 8) return set_err(OBG_EINVAL, "levels must be in 1..8, got %d", levels);
  if (n_trees < 0) return set_err(OBG_EINVAL, "n_trees must be >= 0");
  if (n_trees == 0) return OBG_OK;
  if (!pyramids || !cube) return set_err(OBG_EINVAL, "null buffer");
  const int64_t CW = cube_words(levels);
  k_leaf_cube<<<grid_for(CW * n_trees, 256, sm_count() * 8), 256, 0, as_stream(stream)>>>(
      pyramids, pyr_words(levels), levels, n_trees, cube);
  LAUNCH_CHECK("k_leaf_cube");
  return finish_operand(cube, n_trees, levels, as_stream(stream));
}

template <int L, int OUT>
static int launch_classify_flat(const uint8_t* frames, int64_t n_pixels, const uint32_t* cube, uint8_t* mask,
                                unsigned long long* counts, cudaStream_t st, bool dep, const uint32_t* gate = nullptr) {
  constexpr bool SMEM = L <= 6;
  const size_t smem = SMEM ? size_t(SmemC<L>::words) * 4 : 0;
  const int64_t n_units = n_pixels / 16;
  static DevCache bps_cache;                 // per instantiation and device: smem opt-in, occupancy
  int& bps = bps_cache();
  if (bps == 0) {
    CUDA_TRY(cudaFuncSetAttribute(k_classify_flat<L, SMEM, OUT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(smem)));
    bps = occupancy(k_classify_flat<L, SMEM, OUT>, CLS_BLOCK, smem);
  }
  int64_t grid = int64_t(sm_count()) * bps;
  const int64_t need = (n_units + CLS_BLOCK - 1) / CLS_BLOCK;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  cudaError_t le = launch_dep(k_classify_flat<L, SMEM, OUT>, dim3(unsigned(grid)), dim3(CLS_BLOCK), smem, st, dep ? 2 : 0, frames,
                              n_units, n_pixels, cube, mask, counts, gate);
  if (le != cudaSuccess) return set_err(OBG_ECUDA, "launch of k_classify_flat failed: %s", cudaGetErrorString(le));
  LAUNCH_CHECK("k_classify_flat");
  return OBG_OK;
}

template <int OUT>
static int launch_classify_l7(const uint8_t* frames, int64_t n_pixels, const uint32_t* cube, uint8_t* mask,
                              unsigned long long* counts, cudaStream_t st) {
  const size_t smem_s = size_t(S7_WORDS) * 4, smem_c = size_t(C7_WORDS) * 4;
  static DevCache attr;
  if (!attr()) {
    CUDA_TRY(cudaFuncSetAttribute(k_classify_l7<OUT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_s)));
    CUDA_TRY(cudaFuncSetAttribute(k_classify_l7<OUT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_c)));
    attr() = 1;
  }
  const int64_t n_units = n_pixels / 16;
  int64_t grid = sm_count();
  const int64_t need = (n_units + C7_BLOCK - 1) / C7_BLOCK;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  k_classify_l7<OUT, false><<<unsigned(grid), C7_BLOCK, smem_s, st>>>(frames, n_units, n_pixels, cube, mask, counts);
  LAUNCH_CHECK("k_classify_l7<states>");
  k_classify_l7<OUT, true><<<unsigned(grid), C7_BLOCK, smem_c, st>>>(frames, n_units, n_pixels, cube, mask, counts);
  LAUNCH_CHECK("k_classify_l7<cube>");
#if OBG_L7_CELLS
  // third candidate: every occupied L=6 cell is full, so the L=6 kernel on the
  // full-cell bitset gives the same masks at the L=6 kernel's speed
  return launch_classify_flat<6, OUT>(frames, n_pixels, cube + S7_CELLS_OFF, mask, counts, st, false,
                                      cube + S7_COUNTS_OFF);
#else
  return OBG_OK;
#endif
}

// obg_classify / obg_classify_confusion: `mask` is the output mask or the
// truth mask (OUT_CONF_*), packed = bit-packed layout.
template <int OUT>
static int classify_dispatch(const uint8_t* frames, int n_frames, int height, int width, int levels, int grid_rows,
                             int grid_cols, const uint32_t* cube_bits, uint8_t* mask, unsigned long long* counts,
                             cudaStream_t st, bool dep = false) {
  constexpr bool packed = OUT == OUT_PACKED || OUT == OUT_CONF_PACKED;
  const int64_t P = int64_t(height) * width;
  const int64_t n_pixels = P * n_frames;
  const bool aligned = (reinterpret_cast<uintptr_t>(frames) % 16) == 0 &&
                       (reinterpret_cast<uintptr_t>(mask) % (packed ? 2 : 16)) == 0;
  const bool flat = grid_rows == 1 && grid_cols == 1 && aligned && (!packed || (P % 16) == 0);
  if (flat) {
    switch (levels) {
      case 1: return launch_classify_flat<1, OUT>(frames, n_pixels, cube_bits, mask, counts, st, dep);
      case 2: return launch_classify_flat<2, OUT>(frames, n_pixels, cube_bits, mask, counts, st, dep);
      case 3: return launch_classify_flat<3, OUT>(frames, n_pixels, cube_bits, mask, counts, st, dep);
      case 4: return launch_classify_flat<4, OUT>(frames, n_pixels, cube_bits, mask, counts, st, dep);
      case 5: return launch_classify_flat<5, OUT>(frames, n_pixels, cube_bits, mask, counts, st, dep);
      case 6: return launch_classify_flat<6, OUT>(frames, n_pixels, cube_bits, mask, counts, st, dep);
      case 7: return launch_classify_l7<OUT>(frames, n_pixels, cube_bits, mask, counts, st);
      default: return launch_classify_flat<8, OUT>(frames, n_pixels, cube_bits, mask, counts, st, dep);
    }
  }
  const bool band = (grid_rows > 1 || grid_cols > 1) && levels <= 6 && (width % 16) == 0 && aligned &&
                    grid_cols <= 16 && grid_rows <= height &&
                    size_t(grid_cols) * 4 * (levels == 6 ? BandOp<6>::OPW : BandOp<5>::OPW) <= 227 * 1024;
  if (band) {
    switch (levels) {
      case 1: return launch_classify_band<1, OUT>(frames, n_frames, height, width, grid_rows, grid_cols, cube_bits, mask, counts, st);
      case 2: return launch_classify_band<2, OUT>(frames, n_frames, height, width, grid_rows, grid_cols, cube_bits, mask, counts, st);
      case 3: return launch_classify_band<3, OUT>(frames, n_frames, height, width, grid_rows, grid_cols, cube_bits, mask, counts, st);
      case 4: return launch_classify_band<4, OUT>(frames, n_frames, height, width, grid_rows, grid_cols, cube_bits, mask, counts, st);
      case 5: return launch_classify_band<5, OUT>(frames, n_frames, height, width, grid_rows, grid_cols, cube_bits, mask, counts, st);
      default: return launch_classify_band<6, OUT>(frames, n_frames, height, width, grid_rows, grid_cols, cube_bits, mask, counts, st);
    }
  }
  const int64_t threads = ((P + 7) / 8) * n_frames;
  const int grid = grid_for(threads, 256, sm_count() * 8);
  k_classify_generic<OUT><<<grid, 256, 0, st>>>(frames, n_frames, height, width, levels, grid_rows, grid_cols,
                                                cube_bits, mask, counts);
  LAUNCH_CHECK("k_classify_generic");
  return OBG_OK;
}

static int classify_args(int n_frames, int height, int width, int levels, int grid_rows, int grid_cols,
                         int mask_format) {
  if (levels < 1 || levels > 8) return set_err(OBG_EINVAL, "levels must be in 1..8, got %d", levels);
  if (n_frames < 0) return set_err(OBG_EINVAL, "n_frames must be >= 0");
  if (height < 1 || width < 1) return set_err(OBG_EINVAL, "frame dimensions must be >= 1");
  if (grid_rows < 1 || grid_cols < 1) return set_err(OBG_EINVAL, "grid dimensions must be >= 1");
  if (mask_format != OBG_MASK_U8 && mask_format != OBG_MASK_PACKED)
    return set_err(OBG_EINVAL, "unknown mask_format %d", mask_format);
  return OBG_OK;
}

int obg_classify(const uint8_t* frames, int n_frames, int height, int width, int levels, int grid_rows, int grid_cols,
                 const uint32_t* cube_bits, uint8_t* mask, int mask_format, void* stream) {
  g_err[0] = 0;
  const bool dep = (mask_format & OBG_MASK_AFTER_MODEL) != 0;      // launched as a dependent of the model build
  mask_format &= ~OBG_MASK_AFTER_MODEL;
  if (int rc = classify_args(n_frames, height, width, levels, grid_rows, grid_cols, mask_format)) return rc;
  if (n_frames == 0) return OBG_OK;
  if (!frames || !cube_bits || !mask) return set_err(OBG_EINVAL, "null buffer");
  cudaStream_t st = as_stream(stream);
  if (mask_format == OBG_MASK_PACKED)
    return classify_dispatch<OUT_PACKED>(frames, n_frames, height, width, levels, grid_rows, grid_cols, cube_bits,
                                         mask, nullptr, st, dep);
  return classify_dispatch<OUT_U8>(frames, n_frames, height, width, levels, grid_rows, grid_cols, cube_bits, mask,
                                   nullptr, st, dep);
}

int obg_classify_confusion(const uint8_t* frames, int n_frames, int height, int width, int levels, int grid_rows,
                           int grid_cols, const uint32_t* cube_bits, const uint8_t* truth, int truth_format,
                           uint64_t* counts, void* stream) {
  g_err[0] = 0;
  if (int rc = classify_args(n_frames, height, width, levels, grid_rows, grid_cols, truth_format)) return rc;
  if (n_frames == 0) return OBG_OK;
  if (!frames || !cube_bits || !truth || !counts) return set_err(OBG_EINVAL, "null buffer");
  cudaStream_t st = as_stream(stream);
  uint8_t* t = const_cast<uint8_t*>(truth);                  // read only (OUT_CONF_*)
  unsigned long long* c = reinterpret_cast<unsigned long long*>(counts);
  if (truth_format == OBG_MASK_PACKED)
    return classify_dispatch<OUT_CONF_PACKED>(frames, n_frames, height, width, levels, grid_rows, grid_cols,
                                              cube_bits, t, c, st);
  return classify_dispatch<OUT_CONF_U8>(frames, n_frames, height, width, levels, grid_rows, grid_cols, cube_bits, t,
                                        c, st);
}

// ---------------------------------------------------------------------------
// Host frames in, host masks out in ONE call: the reference's own
// detect_octree(model, frame) signature (detect.py:22-53; numpy in, numpy bool
// out), which the reference CLI loops over frame by frame (cli.py:181-187,
// 262-288).  A pageable cudaMemcpy of a 6.2 MB frame runs at ~12 GB/s (the
// driver's single-threaded staging copy); here the frame is copied into
// pinned staging by libobg's host copy pool in two halves, each half's H2D
// starting as soon as it is staged, the classify kernel follows on the same
// stream, and the mask comes back through pinned staging in two halves, the
// first copied out to the caller while the second is still in flight.
// Staging and device buffers are cached per host thread (grown on demand,
// released by obg_host_stage_release).
// ---------------------------------------------------------------------------
namespace {
struct HostStage {
  int device = -1;
  uint8_t *pin_in = nullptr, *pin_out = nullptr, *dev_in = nullptr, *dev_out = nullptr;
  size_t in_cap = 0, out_cap = 0;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  void release() {
    if (pin_in) cudaFreeHost(pin_in);
    if (pin_out) cudaFreeHost(pin_out);
    if (dev_in) cudaFree(dev_in);
    if (dev_out) cudaFree(dev_out);
    for (auto& e : ev)
      if (e) { cudaEventDestroy(e); e = nullptr; }
    pin_in = pin_out = dev_in = dev_out = nullptr;
    in_cap = out_cap = 0;
    device = -1;
  }
};
thread_local HostStage g_stage;

int stage_reserve(HostStage& s, size_t in_bytes, size_t out_bytes) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if (s.device != dev) s.release();
  s.device = dev;
  for (auto& e : s.ev)
    if (!e) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  if (s.in_cap < in_bytes) {
    if (s.pin_in) cudaFreeHost(s.pin_in);
    if (s.dev_in) cudaFree(s.dev_in);
    s.pin_in = s.dev_in = nullptr;
    s.in_cap = 0;
    CUDA_TRY(cudaMallocHost(&s.pin_in, in_bytes));
    CUDA_TRY(cudaMalloc(&s.dev_in, in_bytes));
    s.in_cap = in_bytes;
  }
  if (s.out_cap < out_bytes) {
    if (s.pin_out) cudaFreeHost(s.pin_out);
    if (s.dev_out) cudaFree(s.dev_out);
    s.pin_out = s.dev_out = nullptr;
    s.out_cap = 0;
    CUDA_TRY(cudaMallocHost(&s.pin_out, out_bytes));
    CUDA_TRY(cudaMalloc(&s.dev_out, out_bytes));
    s.out_cap = out_bytes;
  }
  return OBG_OK;
}

int pool_copy(uint8_t* dst, const uint8_t* src, int64_t bytes, bool to_pinned) {
  return obg_host_copy(src, bytes, dst, to_pinned ? 1 : 0);
}
}  // namespace

void obg_host_stage_release(void) { g_stage.release(); }

int obg_detect_host(const uint8_t* frames, int n_frames, int height, int width, int levels, int grid_rows,
                    int grid_cols, const uint32_t* cube_bits, uint8_t* mask, void* stream) {
  g_err[0] = 0;
  if (int rc = classify_args(n_frames, height, width, levels, grid_rows, grid_cols, OBG_MASK_U8)) return rc;
  if (n_frames == 0) return OBG_OK;
  if (!frames || !cube_bits || !mask) return set_err(OBG_EINVAL, "null buffer");
  cudaStream_t st = as_stream(stream);
  const int64_t P = int64_t(height) * width;
  // frames per pass: at most ~64 MiB of staging
  const int64_t per_pass = std::max<int64_t>(1, std::min<int64_t>(n_frames, (int64_t(64) << 20) / (3 * P)));
  HostStage& s = g_stage;
  if (int rc = stage_reserve(s, size_t(per_pass * 3 * P), size_t(per_pass * P))) return rc;
  static const bool trace = getenv("OBG_DETECT_TRACE") != nullptr;
  auto now = [] { return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  double tq[8] = {0};
  tq[0] = now();
  for (int64_t f0 = 0; f0 < n_frames; f0 += per_pass) {
    const int64_t m = std::min<int64_t>(per_pass, n_frames - f0);
    const int64_t in_bytes = m * 3 * P, out_bytes = m * P;
    const uint8_t* src = frames + f0 * 3 * P;
    uint8_t* dst = mask + f0 * P;
    // in: two halves (cut at a multiple of 256 bytes), stage -> H2D
    // (frames below 1 MiB go as one piece: the second copy call would cost more than the overlap)
    const int64_t cut_in = in_bytes >= (int64_t(1) << 20) ? (in_bytes / 2) & ~int64_t(255) : 0;
    const int64_t in_off[3] = {0, cut_in, in_bytes};
    for (int h = 0; h < 2; ++h) {
      const int64_t len = in_off[h + 1] - in_off[h];
      if (len == 0) continue;
      if (int rc = pool_copy(s.pin_in + in_off[h], src + in_off[h], len, true)) return rc;
      tq[1 + 2 * h] = now();
      CUDA_TRY(cudaMemcpyAsync(s.dev_in + in_off[h], s.pin_in + in_off[h], size_t(len), cudaMemcpyHostToDevice, st));
      tq[2 + 2 * h] = now();
    }
    if (int rc = classify_dispatch<OUT_U8>(s.dev_in, int(m), height, width, levels, grid_rows, grid_cols, cube_bits,
                                           s.dev_out, nullptr, st))
      return rc;
    // out: two halves, D2H -> copy out (the second transfer overlaps the first copy)
    const int64_t cut_out = out_bytes >= (int64_t(1) << 20) ? (out_bytes / 2) & ~int64_t(255) : 0;
    const int64_t out_off[3] = {0, cut_out, out_bytes};
    for (int h = 0; h < 2; ++h) {
      const int64_t len = out_off[h + 1] - out_off[h];
      if (len > 0)
        CUDA_TRY(cudaMemcpyAsync(s.pin_out + out_off[h], s.dev_out + out_off[h], size_t(len), cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaEventRecord(s.ev[h], st));
    }
    tq[5] = now();
    for (int h = 0; h < 2; ++h) {
      CUDA_TRY(cudaEventSynchronize(s.ev[h]));
      if (h == 0) tq[6] = now();
      const int64_t len = out_off[h + 1] - out_off[h];
      if (len > 0)
        if (int rc = pool_copy(dst + out_off[h], s.pin_out + out_off[h], len, false)) return rc;
    }
    tq[7] = now();
    if (trace)
      fprintf(stderr, "obg_detect_host: stage0 %.0f h2d0-call %.0f stage1 %.0f h2d1-call %.0f launch+d2h-calls %.0f wait0 %.0f rest %.0f total %.0f us\n",
              tq[1] - tq[0], tq[2] - tq[1], tq[3] - tq[2], tq[4] - tq[3], tq[5] - tq[4], tq[6] - tq[5], tq[7] - tq[6], tq[7] - tq[0]);
  }
  return OBG_OK;
}

int64_t obg_serialize_workspace_bytes(int levels) {
  if (levels < 1 || levels > 8) return -1;
  const int64_t PW = pyr_words(levels);
  return (PW + 1 + (PW + SCAN_CHUNK - 1) / SCAN_CHUNK + 16) * 4;     // prefix (+ node count), chunk totals
}

int obg_serialize(const uint32_t* pyramid, int levels, int has_root, uint8_t* out, int64_t out_capacity,
                  int64_t* n_out, void* workspace, int64_t workspace_bytes, void* stream) {
  g_err[0] = 0;
  if (levels < 1 || levels > 8) return set_err(OBG_EINVAL, "levels must be in 1..8, got %d", levels);
  if (!pyramid || !n_out) return set_err(OBG_EINVAL, "null buffer");
  if (workspace_bytes < obg_serialize_workspace_bytes(levels) || !workspace)
    return set_err(OBG_EINVAL, "workspace too small");
  cudaStream_t st = as_stream(stream);
  const int64_t PW = pyr_words(levels);
  uint32_t* prefix = static_cast<uint32_t*>(workspace);
  uint32_t* partials = prefix + PW + 1;
  const unsigned chunks = unsigned((PW + SCAN_CHUNK - 1) / SCAN_CHUNK);
  k_scan_partials<<<chunks, SCAN_BLOCK, 0, st>>>(pyramid, PW, partials);
  LAUNCH_CHECK("k_scan_partials");
  k_scan_finish<<<chunks, SCAN_BLOCK, 0, st>>>(pyramid, PW, partials, prefix);
  LAUNCH_CHECK("k_scan_finish");
  uint32_t h_nodes = 0;
  CUDA_TRY(cudaMemcpyAsync(&h_nodes, prefix + PW, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  const int64_t nodes = h_nodes;
  if (!has_root && nodes == 0) { *n_out = 0; return OBG_OK; }
  const int64_t total = nodes + 1;
  *n_out = total;
  if (!out || out_capacity < total)
    return set_err(OBG_EINVAL, "output capacity %lld < %lld bytes", (long long)out_capacity, (long long)total);
  // root byte: the level-1 child mask
  CUDA_TRY(cudaMemcpyAsync(out, pyramid, 1, cudaMemcpyDeviceToDevice, st));
  if (nodes > 0) {
    k_serialize<<<grid_for(PW * 32, 256, sm_count() * 16), 256, 0, st>>>(pyramid, prefix, levels, out);
    LAUNCH_CHECK("k_serialize");
  }
  return OBG_OK;
}


// ---------------------------------------------------------------------------
// comparison baselines (detect.py:56-83)
// ---------------------------------------------------------------------------
int obg_frame_diff(const uint8_t* prev, const uint8_t* cur, int n_pairs, int64_t pixels, int diff_threshold,
                   uint8_t* masks, void* stream) {
  g_err[0] = 0;
  if (n_pairs < 0) return set_err(OBG_EINVAL, "n_pairs must be >= 0");
  if (pixels < 0) return set_err(OBG_EINVAL, "pixels must be >= 0");
  if (n_pairs == 0 || pixels == 0) return OBG_OK;
  if (!prev || !cur || !masks) return set_err(OBG_EINVAL, "null buffer");
  cudaStream_t st = as_stream(stream);
  const bool aligned = (pixels % 16) == 0 && (reinterpret_cast<uintptr_t>(prev) % 16) == 0 &&
                       (reinterpret_cast<uintptr_t>(cur) % 16) == 0 && (reinterpret_cast<uintptr_t>(masks) % 16) == 0;
  if (!aligned) {
    const int64_t total = int64_t(n_pairs) * pixels;
    k_frame_diff_px<<<grid_for(total, FD_BLOCK, sm_count() * 16), FD_BLOCK, 0, st>>>(prev, cur, n_pairs, pixels,
                                                                                    diff_threshold, masks);
    LAUNCH_CHECK("k_frame_diff_px");
    return OBG_OK;
  }
  const int mode = diff_threshold < 0 ? 1 : diff_threshold >= 255 ? 2 : 0;
  const int seq = cur == prev + 3 * pixels ? 1 : 0;
  const int64_t n_units = pixels / 16;
  // chunks of consecutive pairs per thread: enough items to fill the GPU
  // (about 8 units per SM thread slot), long chunks otherwise
  const int64_t want = int64_t(sm_count()) * 2048 * 2;
  int64_t c = (n_units * n_pairs) / (want > 0 ? want : 1);
  if (c > n_pairs) c = n_pairs;
  if (c < 1) c = 1;
  int chunk = int(c);
  if (!seq) chunk = 1;
  const int64_t items = n_units * ((n_pairs + chunk - 1) / chunk);
  k_frame_diff<<<grid_for(items, FD_BLOCK, sm_count() * 16), FD_BLOCK, 0, st>>>(prev, cur, n_pairs, pixels, n_units,
                                                                               chunk, diff_threshold, mode, seq, masks);
  LAUNCH_CHECK("k_frame_diff");
  return OBG_OK;
}

int obg_running_average(const uint8_t* frames, int n_frames, int64_t pixels, int64_t frames_seen, double* average,
                        int diff_threshold, uint8_t* masks, void* stream) {
  g_err[0] = 0;
  if (n_frames < 0) return set_err(OBG_EINVAL, "n_frames must be >= 0");
  if (pixels < 0) return set_err(OBG_EINVAL, "pixels must be >= 0");
  if (n_frames == 0 || pixels == 0) return OBG_OK;
  if (!frames || !average || !masks) return set_err(OBG_EINVAL, "null buffer");
  cudaStream_t st = as_stream(stream);
  k_running_average<<<grid_for(pixels, FD_BLOCK, sm_count() * 16), FD_BLOCK, 0, st>>>(
      frames, n_frames, pixels, frames_seen, average, double(diff_threshold), masks);
  LAUNCH_CHECK("k_running_average");
  return OBG_OK;
}

// ---------------------------------------------------------------------------
// Sharded model build (distributed.py): the cube-order
// build + per-node tree counts of this rank's frames; after an all-reduce of
// the counts, the threshold + path-order conversion.
// ---------------------------------------------------------------------------
static int64_t merge_blocks(int levels) {
  int64_t blocks = 1;
  for (int l = 3; l <= levels; ++l) blocks += mf_blocks(l);
  return blocks;
}

int obg_build_counts(const uint8_t* frames, int n_frames, int height, int width, int levels, int grid_rows,
                     int grid_cols, int group_size, uint32_t* counts, void* workspace, int64_t workspace_bytes,
                     int flags, void* stream) {
  g_err[0] = 0;
  if (levels < 1 || levels > 8) return set_err(OBG_EINVAL, "levels must be in 1..8, got %d", levels);
  if (!counts) return set_err(OBG_EINVAL, "null buffer");
  const int64_t n_regions = int64_t(grid_rows) * grid_cols;
  if (n_regions > 65535) return set_err(OBG_EUNSUPPORTED, "too many regions (%lld > 65535)", (long long)n_regions);
  // tree_pyramids: K1's leading-word clears need a target; the counts buffer
  // is fully overwritten afterwards, so it doubles as that scratch
  int rc = build_presence_impl(frames, n_frames, height, width, levels, grid_rows, grid_cols, group_size, counts,
                               nullptr, workspace, workspace_bytes, flags, nullptr, 0, stream, /*cube_levels=*/true);
  if (rc != OBG_OK) return rc;
  cudaStream_t st = as_stream(stream);
  const int n_groups = n_frames / group_size;
  k_merge_fused<1><<<dim3(unsigned(merge_blocks(levels)), unsigned(n_regions)), dim3(32, MERGE_GROUPS_C), 0, st>>>(
      static_cast<uint32_t*>(workspace), n_groups, int(n_regions), levels, 0, nullptr, nullptr, counts);
  LAUNCH_CHECK("k_merge_fused<count>");
  return OBG_OK;
}

int obg_threshold_counts(const uint32_t* counts, int n_regions, int levels, int64_t k_min, uint32_t* out_merged,
                         uint32_t* out_cube, void* stream) {
  g_err[0] = 0;
  if (levels < 1 || levels > 8) return set_err(OBG_EINVAL, "levels must be in 1..8, got %d", levels);
  if (n_regions < 1 || n_regions > 65535) return set_err(OBG_EINVAL, "n_regions must be in 1..65535");
  if (k_min < 1) return set_err(OBG_EINVAL, "k_min must be >= 1, got %lld", (long long)k_min);
  if (!counts || !out_merged || !out_cube) return set_err(OBG_EINVAL, "null buffer");
  cudaStream_t st = as_stream(stream);
  k_merge_fused<2><<<dim3(unsigned(merge_blocks(levels)), unsigned(n_regions)), dim3(32, MERGE_GROUPS_C), 0, st>>>(
      nullptr, 0, n_regions, levels, k_min, out_cube, out_merged, const_cast<uint32_t*>(counts));
  LAUNCH_CHECK("k_merge_fused<threshold>");
  return finish_operand(out_cube, n_regions, levels, st);
}
