// One translation unit per compile-time FFT length: build.py compiles this
// file once per length with -DVK_LEN=N (the lengths' kernels are the bulk of
// the build and compile in parallel).  Variant choices per length come from
// B200 measurements (see the comments).
#include "fast_entry.cuh"

#ifndef VK_LEN
#error "compile with -DVK_LEN=<fft length>"
#endif

namespace vk {

#if VK_LEN == 64
FastEntry fast_entry_64() { return make_entry<8, 8, 16, 16, false, true, 1, false, false, true, 1, true, 2, 8, 0, true>(); }  // 64 (FRC half grids, small z)
#elif VK_LEN == 96
FastEntry fast_entry_96() { return make_entry<8, 12, 16, 16, false, true, 1, false, false, true, 1, true, 2, 8, 6, true>(); }  // 96 (z: TMA 6; y bulk L=8)
#elif VK_LEN == 144
FastEntry fast_entry_144() { return make_entry<12, 12, 16, 16, false, true, 1, false, true, false, 8, true, 2, 8, 6, true>(); }  // 144 (z: TMA 6; y bulk L=8)
#elif VK_LEN == 192
FastEntry fast_entry_192() { return make_entry<12, 16, 16, 16, false, true, 1, false, true, false, 5, true, 2, 8, 4, true>(); }  // 192 (z: TMA tile, 4 CTAs/SM; y bulk L=8)
#elif VK_LEN == 256
FastEntry fast_entry_256() { return make_entry<16, 16, 16, 16, false, true, 1, false, false, true, 1, true, 2, 8, 0, true>(); }  // 256 (y bulk L=8)
#elif VK_LEN == 288
// 288: TMA-staged x pass (C1 x passes 0.0730 vs 0.0753 ms per iteration; at
// 576 it loses: profiles/r01/final/xtma.log)
// x pass with a 3-CTA register floor: the packed complex arithmetic took the
// staged kernel from 72 to 75 registers, i.e. from 3 to 2 resident CTAs
// (C1 x passes +13%, profiles/r02/final)
// 8 lines per CTA (1326 CTAs on the C1 grid instead of 702 at 3 per SM, i.e.
// ~1.5 waves at 6 per SM instead of 1.6 at 3 with a 58%-full tail): C1 +2.0%,
// C3 +1.8% (profiles/r02/x288_l8_ab.txt; a 5-CTA register floor without
// the 32-byte stack measured the same).
FastEntry fast_entry_288() { return make_entry<16, 18, 8, 16, false, true, 6, false, false, true, 1, true, 2, 8, 0, true, true>(); }  // 288 (y: bulk, L=8)
#elif VK_LEN == 576
#if defined(VK_X576_VARIANT) && VK_X576_VARIANT == 1  // experiment: 16-line x pass (32 rows, 256-byte pieces), 2 CTAs/SM
FastEntry fast_entry_576() { return make_entry<24, 24, 16, 8, true, true, 2, false, false, true, 1, true, 2, 8, 0, true>(); }
#elif defined(VK_X576_VARIANT) && VK_X576_VARIANT == 2  // the same with TMA-staged spectrum rows
FastEntry fast_entry_576() { return make_entry<24, 24, 16, 8, true, true, 2, false, false, true, 1, true, 2, 8, 0, true, true>(); }
#else
FastEntry fast_entry_576() { return make_entry<24, 24, 8, 8, true, true, 5, false, false, true, 1, true, 2, 0, 0, true>(); }  // 576: global twiddles -> 5 x/y CTAs/SM (y L=4: slower); y bulk copies
#endif
#elif VK_LEN == 1080
// 1080: TMA-staged x pass with a 2-CTA register floor (96 regs, 80 B stack;
// without the floor the staged loads take 129 registers and 1 CTA/SM): C4
// 2.884 vs 2.940 ms per iteration (profiles/r01/final/x1080.log)
// y pass: 4 lines per CTA (C4 3.59e10; 2 lines 3.47e10, 8 lines 3.11e10:
// profiles/r02/y1080_lines_ab.txt)
FastEntry fast_entry_1080() { return make_entry<30, 36, 8, 4, false, true, 2, true, false, true, 1, true, 2, 4, 0, true, true>(); }  // 1080 (Ix = 1000: partial chunks are common)
#elif VK_LEN == 2160
// 2160: no smem twiddles / OTF tile -> 2 CTAs per SM; no PDL (CTAs parked
// in griddepcontrol.wait would hold the scarce slots the batch lanes'
// kernels need: C5 3.05e10 without vs 2.66e10 with, profiles/r01/pdl.log)
// and the TMA-staged x pass with a 2-CTA register floor (168 regs, 48 B
// stack): C5 x passes 0.0774 vs 0.0801 ms per field-iteration (final/x2160.log)
FastEntry fast_entry_2160() { return make_entry<45, 48, 4, 2, true, false, 2, false, false, true, 1, false, 2, 2, 0, true, true>(); }  // y L=2
#else
// Any other even 5-smooth length with a two-pass split R1 x R2 (R1 <= R2 <= 48):
// the variant choices follow the measured entries above by size class
// (lines per CTA from shared memory, twiddles from global for long lines,
// a TMA z tile with a resident-CTA floor up to 256 points, PDL except at
// 2160-class lengths).
namespace gen {
constexpr int isqrt(int n) {
  int r = 0;
  while ((r + 1) * (r + 1) <= n) ++r;
  return r;
}
constexpr int r1(int n) {
  for (int d = isqrt(n); d > 1; --d)
    if (n % d == 0) return d;
  return 1;
}
constexpr int N = VK_LEN, R1 = r1(N), R2 = N / R1;
static_assert(R1 > 1 && R2 <= 48, "VK_LEN needs a two-pass split with radices <= 48");
constexpr int LX = N <= 640 ? 8 : N <= 1280 ? 4 : 2;
constexpr int LZ = N <= 256 ? 16 : LX;
constexpr bool TWG = (LX == 8 && N >= 512) || N >= 1500;
constexpr bool ZTWG = N >= 128;
constexpr int cmin(int a, int b) { return a < b ? a : b; }
constexpr int NTZ = (16 * R2 + 31) / 32 * 32;
// TMA z tile: resident CTAs by shared memory, capped at 6 and at >= 56 registers per thread
constexpr int ZFLOOR = LZ == 16 ? cmin(cmin(6, 200 * 1024 / (2 * N * 16 * 8 + (ZTWG ? 0 : N * 8))), 65536 / (NTZ * 56))
                                : 0;
}  // namespace gen
#define VK_CAT2(a, b) a##b
#define VK_CAT(a, b) VK_CAT2(a, b)
FastEntry VK_CAT(fast_entry_, VK_LEN)() {
  using namespace gen;
  return make_entry<R1, R2, LX, LZ, TWG, (N <= 640), (LX <= 2 ? 2 : 1), (LX <= 4), ZTWG, (N < 128), 1, (N < 2000), 2,
                    0, ZFLOOR, true, false>();
}
#endif

}  // namespace vk
