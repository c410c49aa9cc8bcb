// numpy-compatible PCG64 stream with O(log n) jump-ahead, used to reproduce
// `rng.choice(n, 3, replace=False)` (posest.py:243,252) bit-exactly on device.
//
// Third-party algorithm: numpy 2.3.5 (random/_pcg64, Generator.choice with
// Floyd's algorithm + tail shuffle, Lemire bounded draws with rejection).
// See oracle/rng.py for the CPU restatement this is tested against.
//
// The uint32 stream of a generator is addressed by position p (number of
// 32-bit words consumed since the stored state).  Word p comes from 64-bit
// output m = (p - has0) >> 1 (low half first), i.e. from the state after
// m + 1 LCG steps — reachable in O(log m) with the classic LCG jump.
#pragma once
#include <cstdint>
#include "vl_common.cuh"

namespace vl {

typedef unsigned __int128 u128;

VL_HD u128 pcg_mult() {
  return (((u128)0x2360ED051FC65DA4ull) << 64) | (u128)0x4385DF649FCCF645ull;
}

VL_HD uint64_t pcg_out(u128 s) {
  const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  const uint64_t x = hi ^ lo;
  const unsigned rot = (unsigned)(s >> 122);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

// state after `delta` LCG steps.
VL_HD u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
  u128 cur_mult = pcg_mult(), cur_plus = inc;
  u128 acc_mult = 1, acc_plus = 0;
  while (delta > 0) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

struct GenState {
  u128 state, inc;
  uint32_t has0, uint0;
};

// Sequential word reader positioned anywhere in the uint32 stream.
struct WordReader {
  u128 st;        // state after the 64-bit output currently buffered
  u128 inc;
  uint64_t cur;   // current 64-bit output
  int half;       // 0: next word is low half of cur (needs no step), 1: high half, 2: need step
  int pending0;   // the stored buffered word is next
  uint32_t buf0;

  VL_HD void init(const GenState& g, uint64_t pos) {
    inc = g.inc;
    pending0 = 0;
    buf0 = g.uint0;
    if (g.has0) {
      if (pos == 0) {
        pending0 = 1;
        st = g.state;
        half = 2;
        return;
      }
      pos -= 1;
    }
    const uint64_t m = pos >> 1;
    st = pcg_advance(g.state, g.inc, m + 1);
    cur = pcg_out(st);
    half = (int)(pos & 1);
  }
  VL_HD uint32_t next() {
    if (pending0) {
      pending0 = 0;
      return buf0;
    }
    if (half == 2) {
      st = st * pcg_mult() + inc;
      cur = pcg_out(st);
      half = 0;
    }
    uint32_t r = (half == 0) ? (uint32_t)cur : (uint32_t)(cur >> 32);
    half = (half == 0) ? 1 : 2;
    return r;
  }
};

// Jump table for a block: tmul[k], tplus[k] advance the LCG by 2^k steps
// (the squarings pcg_advance repeats for every call, done once).
constexpr int kJumpBits = 16;

VL_HD void pcg_jump_table(u128 inc, u128* tmul, u128* tplus) {
  u128 m = pcg_mult(), c = inc;
  for (int k = 0; k < kJumpBits; ++k) {
    tmul[k] = m;
    tplus[k] = c;
    c = (m + 1) * c;
    m *= m;
  }
}

// state after `delta` (< 2^kJumpBits) more LCG steps, from the table: one
// affine composition per set bit of delta (same result as pcg_advance).
VL_HD u128 pcg_advance_tab(u128 state, uint64_t delta, const u128* tmul, const u128* tplus) {
  u128 acc_mult = 1, acc_plus = 0;
  for (int k = 0; delta; ++k, delta >>= 1)
    if (delta & 1) {
      acc_mult *= tmul[k];
      acc_plus = acc_plus * tmul[k] + tplus[k];
    }
  return acc_mult * state + acc_plus;
}

// WordReader positioned at word `pos` from a shared base: base_st is the
// state after 64-bit output m0 + 1 steps, i.e. pcg_advance(g.state, g.inc,
// m0 + 1) with m0 = word index of the batch's first (non-buffered) word >> 1;
// the reader's own output index m >= m0 is then at most a few thousand
// outputs ahead (pos - batch start < 2^kJumpBits words).
VL_HD void reader_init_from(WordReader& rd, const GenState& g, uint64_t pos, u128 base_st, uint64_t m0,
                            const u128* tmul, const u128* tplus) {
  rd.inc = g.inc;
  rd.pending0 = 0;
  rd.buf0 = g.uint0;
  if (g.has0) {
    if (pos == 0) {
      rd.pending0 = 1;
      rd.st = g.state;
      rd.half = 2;
      return;
    }
    pos -= 1;
  }
  const uint64_t m = pos >> 1;
  rd.st = pcg_advance_tab(base_st, m - m0, tmul, tplus);
  rd.cur = pcg_out(rd.st);
  rd.half = (int)(pos & 1);
}

// Number of 32-bit draws one choice(n,3) takes when no rejection happens.
VL_HD int draws_per_sample(int64_t n) { return n == 3 ? 4 : 5; }

// One choice(n,3).  exact=false: speculative, returns false as soon as a
// Lemire rejection would be needed (the caller re-runs exactly).
// exact=true: follows the rejection loop; *used receives the words consumed.
VL_HD bool choice3(WordReader& rd, uint32_t n, bool exact, int64_t* out, int* used) {
  int cnt = 0;
  uint32_t v[3];
  auto bounded = [&](uint32_t j, uint32_t& res) -> bool {
    if (j == 0) {
      res = 0;
      return true;
    }
    const uint32_t excl = j + 1u;
    uint64_t m = (uint64_t)rd.next() * excl;
    ++cnt;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
      const uint32_t thr = (0xFFFFFFFFu - j) % excl;
      while (left < thr) {
        if (!exact) return false;
        m = (uint64_t)rd.next() * excl;
        ++cnt;
        left = (uint32_t)m;
      }
    }
    res = (uint32_t)(m >> 32);
    return true;
  };
  for (int k = 0; k < 3; ++k) {
    const uint32_t j = n - 3u + (uint32_t)k;
    uint32_t val;
    if (!bounded(j, val)) return false;
    bool taken = false;
    for (int i = 0; i < k; ++i) taken |= (v[i] == val);
    v[k] = taken ? j : val;
  }
  for (int i = 2; i >= 1; --i) {
    uint32_t kk;
    if (!bounded((uint32_t)i, kk)) return false;
    const uint32_t tmp = v[kk];
    v[kk] = v[i];
    v[i] = tmp;
  }
  out[0] = v[0];
  out[1] = v[1];
  out[2] = v[2];
  if (used) *used = cnt;
  return true;
}

// ---- numpy SeedSequence(seed).generate_state(4, uint64) -> PCG64 seeding (host)
inline GenState seed_pcg64(uint64_t seed) {
  const uint32_t INIT_A = 0x43B0D7E5u, MULT_A = 0x931E8875u, INIT_B = 0x8B51F9DDu,
                 MULT_B = 0x58F38DEDu, MIX_L = 0xCA01F9DDu, MIX_R = 0x4973F715u;
  uint32_t ent[2];
  int ne = 0;
  ent[ne++] = (uint32_t)seed;
  if (seed >> 32) ent[ne++] = (uint32_t)(seed >> 32);
  uint32_t hc = INIT_A;
  auto hashmix = [&](uint32_t v) {
    v ^= hc;
    hc *= MULT_A;
    v *= hc;
    return v ^ (v >> 16);
  };
  auto mix = [&](uint32_t x, uint32_t y) {
    uint32_t r = MIX_L * x - MIX_R * y;
    return r ^ (r >> 16);
  };
  uint32_t pool[4];
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < ne ? ent[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
  uint32_t w32[8];
  uint32_t hb = INIT_B;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i % 4] ^ hb;
    hb *= MULT_B;
    v *= hb;
    w32[i] = v ^ (v >> 16);
  }
  uint64_t w64[4];
  for (int i = 0; i < 4; ++i) w64[i] = (uint64_t)w32[2 * i] | ((uint64_t)w32[2 * i + 1] << 32);
  const u128 initstate = ((u128)w64[0] << 64) | w64[1];
  const u128 initseq = ((u128)w64[2] << 64) | w64[3];
  GenState g;
  g.inc = (initseq << 1) | 1;
  u128 s = g.inc;  // 0 * M + inc
  s += initstate;
  s = s * pcg_mult() + g.inc;
  g.state = s;
  g.has0 = 0;
  g.uint0 = 0;
  return g;
}

}  // namespace vl
