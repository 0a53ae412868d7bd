// SSMM host dispatch: (NT, NW, MS, REP) -> kernel instantiation.
#include "ssmm_pair.cuh"

namespace smy {

extern template smy_status launch_t<16,1,2,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<32,1,2,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<64,1,2,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<128,1,2,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<SMY_NT_WIDE,1,2,1>(const SsmmArgs&, cudaStream_t);
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
extern template smy_status launch_t<16,1,2,1,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<32,1,2,1,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<64,1,2,1,1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_t<128,1,2,1,1>(const SsmmArgs&, cudaStream_t);

extern template smy_status launch_pair_t<64, 2, 2, 0>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_pair_t<112, 2, 2, 0>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_pair_t<128, 1, 2, 0>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_pair_t<SMY_NT_WIDE, 1, 2, 0>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_pair_t<SMY_NT_WIDE, 1, 2, 1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_pair_t<128, 1, 2, 1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_pair_t<224, 2, 1, 1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_pair_t<SMY_MTP_NT, 2, 2, 1>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_pair_t<128, 1, 1, 0>(const SsmmArgs&, cudaStream_t);
extern template smy_status launch_pair_t<256, 1, 1, 0>(const SsmmArgs&, cudaStream_t);

namespace {
struct Entry { int nt, nw, ms, rep; smy_status (*fn)(const SsmmArgs&, cudaStream_t); int xp = 0; };
const Entry kTable[] = {
    {16, 1, 2, 1, &launch_t<16,1,2,1>},
    {32, 1, 2, 1, &launch_t<32,1,2,1>},
    {64, 1, 2, 1, &launch_t<64,1,2,1>},
    {128, 1, 2, 1, &launch_t<128,1,2,1>},
    {SMY_NT_WIDE, 1, 2, 1, &launch_t<SMY_NT_WIDE,1,2,1>},
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
    // (N, 2N, 32), N > 1: in-smem row expansion, two 128-row halves per m-tile
    {16, 1, 2, 1, &launch_t<16,1,2,1,1>, 1},
    {32, 1, 2, 1, &launch_t<32,1,2,1,1>, 1},
    {64, 1, 2, 1, &launch_t<64,1,2,1,1>, 1},
    {128, 1, 2, 1, &launch_t<128,1,2,1,1>, 1},
};
}  // namespace

bool xp_on(const smy_format& f) { return xp_format(f) && !(debug_flags() & kDebugNoXp); }

int ssmm_pick_nt(int nw, int ms, int rep, int64_t tpg, int xp) {
  // candidate tile widths for this (nw, ms, rep), ascending (xp: the expansion kernels,
  // one weight, two halves)
  if (xp) ms = 2;
  int best = -1, largest = -1;
  for (const Entry& e : kTable) {
    if (e.nw != nw || e.ms != ms || e.rep != rep || e.xp != xp) continue;
    if (e.nt > largest) largest = e.nt;
    if (e.nt >= tpg && (best < 0 || e.nt < best)) best = e.nt;
  }
  return best > 0 ? best : largest;
}

int ssmm_pair_cluster(int nt, int nw, int ms, int rep, int m_tiles, int64_t tokens_per_group, int gather) {
  if (debug_flags() & 16) return 0;  // SMY_DEBUG=16: force the single-CTA kernel
  if (debug_flags() & 32768) gather = 0;  // SMY_DEBUG=32768: pair kernels also for narrow gather tiles
  if (gather && ms == 2 && nw == 1 && nt <= SMY_SINGLE_FAST_GATHER_NT) return 0;
  // an odd m-tile count gives the last pair a phantom peer tile (loads repeated, stores masked)
  if (rep != 1 || m_tiles < 2 || tokens_per_group < 64) return 0;
  if (ms == 2 && !(nw == 2 ? (nt == 64 || nt == 112 || nt == SMY_MTP_NT) : (nt == 128 || nt == SMY_NT_WIDE))) return 0;
  // N == M (plain 2:4): one weight at 128 / 256 tokens, or gate + up (NW = 2) at 224 --
  // two weights per token stage halve the SEL-gather bytes per MMA
  if (ms == 1 && !((nw == 1 && (nt == 128 || nt == 256)) || (nw == 2 && nt == 224))) return 0;
  if (ms != 1 && ms != 2) return 0;
  // (4-CTA clusters sharing weight stages by multicast measured 2x slower on
  // B200 -- probes/mcast_bench.cu -- and were removed)
  return 2;
}

bool ssmm_pair_images_ok(const smy_weight* const* w0, const smy_weight* const* w1, int groups, size_t img_bytes) {
  // the pair kernel addresses every weight image of a launch through ONE tensor map
  // (rows of 128 B, int32 row coordinates): the images must be 128-B aligned
  // relative to each other and span < 256 GB
  uintptr_t lo = UINTPTR_MAX, hi = 0;
  for (int g = 0; g < groups; ++g)
    for (int w = 0; w < 2; ++w) {
      const smy_weight* const* arr = w ? w1 : w0;
      if (!arr) continue;
      const uintptr_t p = reinterpret_cast<uintptr_t>(arr[g]->image);
      if (p < lo) lo = p;
      if (p + img_bytes > hi) hi = p + img_bytes;
    }
  if (hi <= lo) return true;
  for (int g = 0; g < groups; ++g)
    for (int w = 0; w < 2; ++w) {
      const smy_weight* const* arr = w ? w1 : w0;
      if (arr && ((reinterpret_cast<uintptr_t>(arr[g]->image) - lo) & 127)) return false;
    }
  return (hi - lo) / 128 < ((uint64_t)1 << 31);
}

smy_status ssmm_launch_pair(const SsmmArgs& a0, int nt, int nw, int ms, int cl, cudaStream_t s) {
  SsmmArgs a = a0;
  a.debug = debug_flags();
  a.prof = (a.debug & 128) ? debug_prof_buffer(148) : nullptr;
  if (cl != 2 || a.planes != (ms == 2 ? 1 : 0) || (a.block & 127)) {
    set_last_error("ssmm: pair kernel needs (N,M) = (1,2) or N == M tiles of 128-B rows");
    return SMY_E_CONFIG;
  }
  // one tensor map over every weight image of the launch (rows of 128 B)
  uintptr_t lo = UINTPTR_MAX, hi = 0;
  const size_t img_bytes = (size_t)a.m_tiles * a.k_stages * a.block;
  for (int g = 0; g < a.num_groups; ++g)
    for (int w = 0; w < nw; ++w) {
      const uintptr_t p = reinterpret_cast<uintptr_t>(w ? a.img1[g] : a.img0[g]);
      if (!p) continue;
      if (p < lo) lo = p;
      if (p + img_bytes > hi) hi = p + img_bytes;
    }
  if (hi <= lo) return SMY_OK;
  for (int g = 0; g < a.num_groups; ++g)
    for (int w = 0; w < nw; ++w) {
      const uintptr_t p = reinterpret_cast<uintptr_t>(w ? a.img1[g] : a.img0[g]);
      if (p && ((p - lo) & 127)) {
        set_last_error("ssmm: weight images must be 128-B aligned");
        return SMY_E_CONFIG;
      }
    }
  if ((hi - lo) / 128 >= ((uint64_t)1 << 31)) {
    set_last_error("ssmm: weight images span more than 256 GB");
    return SMY_E_CONFIG;
  }
  a.wbase = reinterpret_cast<const uint8_t*>(lo);
  smy_status st = make_w_tmap(&a.tmap_w, a.wbase, (int64_t)((hi - lo) / 128), (kABytes + kEBytes + 64 + 127) / 128);
  if (st != SMY_OK) return st;
  if (ms == 2 && nw == 2 && nt == 64) return launch_pair_t<64, 2, 2, 0>(a, s);
  if (ms == 2 && nw == 2 && nt == SMY_MTP_NT && a.mtp_half && a.sel_in) return launch_pair_t<SMY_MTP_NT, 2, 2, 1>(a, s);
  if (ms == 2 && nw == 2 && nt == 112) return launch_pair_t<112, 2, 2, 0>(a, s);
  if (ms == 2 && nw == 1 && nt == 128) return a.sel_in && !(a.debug & 16384) ? launch_pair_t<128, 1, 2, 1>(a, s)
                                                                           : launch_pair_t<128, 1, 2, 0>(a, s);
  // SEL-gathered token rows (gate/up): separate, deeper token ring
  // (SMY_DEBUG=16384: lock-step ring for gather launches too; 262144: split rings for
  // contiguous-row launches too -- ring-structure A/B only)
  if (ms == 2 && nw == 1 && nt == SMY_NT_WIDE)
    return (a.sel_in && !(a.debug & 16384)) || (a.debug & 262144) ? launch_pair_t<SMY_NT_WIDE, 1, 2, 1>(a, s)
                                                                  : launch_pair_t<SMY_NT_WIDE, 1, 2, 0>(a, s);
  if (ms == 1 && nw == 2 && nt == 224) return launch_pair_t<224, 2, 1, 1>(a, s);  // gather launches only
  if (ms == 1 && nw == 1 && nt == 128) return launch_pair_t<128, 1, 1, 0>(a, s);
  if (ms == 1 && nw == 1 && nt == 256) return launch_pair_t<256, 1, 1, 0>(a, s);
  set_last_error("ssmm: unsupported pair (nt, nw)");
  return SMY_E_CONFIG;
}

#ifndef SMY_KSPLIT_MIN_STAGES
#define SMY_KSPLIT_MIN_STAGES 8
#endif
int ssmm_pick_ksplit(int64_t tiles, int k_stages) {
  // Split K so that tiles x splits fills whole waves of the 148 SMs: among the
  // splits that keep >= 8 K-stages per piece and give >= 2 pieces per SM, take
  // the one whose last wave is fullest (work / (waves x 148)), preferring fewer
  // splits on ties (less partial-sum traffic).
  const int64_t sms = 148;
  constexpr int kMin = SMY_KSPLIT_MIN_STAGES;  // K-stages per piece at least
  if (tiles >= 4 * sms || k_stages < 2 * kMin) return 1;
  int best = 1;
  double best_eff = 0.0;
  for (int ks = 1; ks <= k_stages / kMin; ++ks) {
    const int64_t n = tiles * ks;
    if (n < 2 * sms && ks < k_stages / kMin) continue;
    const int64_t waves = (n + sms - 1) / sms;
    const double eff = (double)n / (double)(waves * sms);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best = ks;
    }
  }
  return best;
}

smy_status ssmm_launch(const SsmmArgs& a0, int nt, int nw, int ms, int rep, cudaStream_t s) {
  const SsmmArgs* ap = &a0;
  SsmmArgs dbg;
  if (debug_flags()) {
    dbg = a0;
    dbg.debug = debug_flags();
    dbg.prof = (dbg.debug & 128) ? debug_prof_buffer(148) : nullptr;
    ap = &dbg;
  }
  const SsmmArgs& a = *ap;
  if (a.xp) {
    if (nw != 1 || rep != 1 || a.m_fmt != 2 * a.n_fmt || a.n_fmt < 2) {
      set_last_error("ssmm: the row expansion needs one (N, 2N, 32) weight, N > 1");
      return SMY_E_CONFIG;
    }
    ms = 2;
  }
  for (const Entry& e : kTable)
    if (e.nt == nt && e.nw == nw && e.ms == ms && e.rep == rep && e.xp == a.xp) return e.fn(a, s);
  set_last_error("ssmm: unsupported (nt, nw, ms, rep) combination");
  return SMY_E_CONFIG;
}

}  // namespace smy
