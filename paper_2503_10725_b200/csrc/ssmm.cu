// SSMM host dispatch: (NT, NW, MS, REP) -> kernel instantiation.
#include "ssmm_pair.cuh"

namespace smy {

extern template smy_status launch_t<16,1,2,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<32,1,2,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<64,1,2,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<128,1,2,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<224,1,2,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<16,2,2,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<32,2,2,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<64,2,2,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<112,2,2,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<16,1,1,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<32,1,1,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<64,1,1,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<128,1,1,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<256,1,1,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<16,2,1,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<32,2,1,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<64,2,1,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<128,2,1,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<224,2,1,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<32,1,2,2>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<32,2,2,2>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<32,1,4,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<16,1,8,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<16,1,16,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<32,2,4,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<16,2,8,1>(const SsmmArgs&, cudaStream_t);

extern template smy_status launch_pair_t<64, 2, 2>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_pair_t<112, 2, 2>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_pair_t<128, 1, 2>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_pair_t<224, 1, 2>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_pair_t<112, 2, 4>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_pair_t<224, 1, 4>(const SsmmArgs&, cudaStream_t);

namespace {
struct Entry { int nt, nw, ms, rep; smy_status (*fn)(const SsmmArgs&, cudaStream_t); };
const Entry kTable[] = {
    {16, 1, 2, 1, &launch_t<16,1,2,1>},
    {32, 1, 2, 1, &launch_t<32,1,2,1>},
    {64, 1, 2, 1, &launch_t<64,1,2,1>},
    {128, 1, 2, 1, &launch_t<128,1,2,1>},
    {224, 1, 2, 1, &launch_t<224,1,2,1>},
    {16, 2, 2, 1, &launch_t<16,2,2,1>},
    {32, 2, 2, 1, &launch_t<32,2,2,1>},
    {64, 2, 2, 1, &launch_t<64,2,2,1>},
    {112, 2, 2, 1, &launch_t<112,2,2,1>},
    {16, 1, 1, 1, &launch_t<16,1,1,1>},
    {32, 1, 1, 1, &launch_t<32,1,1,1>},
    {64, 1, 1, 1, &launch_t<64,1,1,1>},
    {128, 1, 1, 1, &launch_t<128,1,1,1>},
    {256, 1, 1, 1, &launch_t<256,1,1,1>},
    {16, 2, 1, 1, &launch_t<16,2,1,1>},
    {32, 2, 1, 1, &launch_t<32,2,1,1>},
    {64, 2, 1, 1, &launch_t<64,2,1,1>},
    {128, 2, 1, 1, &launch_t<128,2,1,1>},
    {224, 2, 1, 1, &launch_t<224,2,1,1>},
    {32, 1, 2, 2, &launch_t<32,1,2,2>},
    {32, 2, 2, 2, &launch_t<32,2,2,2>},
    {32, 1, 4, 1, &launch_t<32,1,4,1>},
    {16, 1, 8, 1, &launch_t<16,1,8,1>},
    {16, 1, 16, 1, &launch_t<16,1,16,1>},
    {32, 2, 4, 1, &launch_t<32,2,4,1>},
    {16, 2, 8, 1, &launch_t<16,2,8,1>},
};
}  // namespace

int ssmm_pick_nt(int nw, int ms, int rep, int64_t tpg) {
  // candidate tile widths for this (nw, ms, rep), ascending
  int best = -1, largest = -1;
  for (const Entry& e : kTable) {
    if (e.nw != nw || e.ms != ms || e.rep != rep) continue;
    if (e.nt > largest) largest = e.nt;
    if (e.nt >= tpg && (best < 0 || e.nt < best)) best = e.nt;
  }
  return best > 0 ? best : largest;
}

int ssmm_pair_cluster(int nt, int nw, int ms, int rep, int m_tiles, int64_t tokens_per_group) {
  if (debug_flags() & 16) return 0;  // SMY_DEBUG=16: force the single-CTA kernel
  if (ms != 2 || rep != 1 || (m_tiles & 1) || tokens_per_group < 64) return 0;
  if (!(nw == 2 ? (nt == 64 || nt == 112) : (nt == 128 || nt == 224))) return 0;
  // two MMA pairs share each weight stage when an expert has >= 2 token tiles
  // (4-CTA multicast clusters measured 2x slower on B200: opt-in via SMY_DEBUG=64)
  const bool quad = (debug_flags() & 64) && tokens_per_group >= 2 * nt && (nt == 112 || nt == 224);
  return quad ? 4 : 2;
}

smy_status ssmm_launch_pair(const SsmmArgs& a0, int nt, int nw, int cl, cudaStream_t s) {
  SsmmArgs a = a0;
  a.debug = debug_flags();
  a.prof = (a.debug & 128) ? debug_prof_buffer(148) : nullptr;
  if (cl == 4 && nw == 2 && nt == 112) return launch_pair_t<112, 2, 4>(a, s);
  if (cl == 4 && nw == 1 && nt == 224) return launch_pair_t<224, 1, 4>(a, s);
  if (nw == 2 && nt == 64) return launch_pair_t<64, 2, 2>(a, s);
  if (nw == 2 && nt == 112) return launch_pair_t<112, 2, 2>(a, s);
  if (nw == 1 && nt == 128) return launch_pair_t<128, 1, 2>(a, s);
  if (nw == 1 && nt == 224) return launch_pair_t<224, 1, 2>(a, s);
  set_last_error("ssmm: unsupported pair (nt, nw)");
  return SMY_E_CONFIG;
}

int ssmm_pick_ksplit(int64_t tiles, int k_stages) {
  // aim for >= 4 tiles per SM while keeping >= 8 K-stages per tile
  const int64_t want = 4 * 148;
  if (tiles >= want || k_stages < 16) return 1;
  int64_t ks = (want + tiles - 1) / tiles;
  if (ks > k_stages / 8) ks = k_stages / 8;
  return ks < 1 ? 1 : (int)ks;
}

smy_status ssmm_launch(const SsmmArgs& a0, int nt, int nw, int ms, int rep, cudaStream_t s) {
  const SsmmArgs* ap = &a0;
  SsmmArgs dbg;
  if (debug_flags()) {
    dbg = a0;
    dbg.debug = debug_flags();
    ap = &dbg;
  }
  const SsmmArgs& a = *ap;
  for (const Entry& e : kTable)
    if (e.nt == nt && e.nw == nw && e.ms == ms && e.rep == rep) return e.fn(a, s);
  set_last_error("ssmm: unsupported (nt, nw, ms, rep) combination");
  return SMY_E_CONFIG;
}

}  // namespace smy
