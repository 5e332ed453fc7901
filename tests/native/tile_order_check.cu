// Host-only check of the pair kernel's wave order (kernels.h: pair_tile_rotation, next_pair_tile):
// for every shape, the pairs' tile sequences partition [0, num_tiles) exactly once, no pair takes
// more tiles than the plain grid stride's busiest pair, and the rotated order meets no more
// distinct M blocks in total than the plain one.  Prints "OK <shapes>" or the first failure.
#include <cstdio>
#include <vector>
#include <set>
#include "../../paper_2407_09577_b200/csrc/kernels.h"

int main() {
  const int Cs[] = {74, 60, 37, 1, 8};
  const int Ks[] = {512, 4096, 8192};
  int shapes = 0;
  for (int C : Cs)
    for (int K : Ks)
      for (int mb = 1; mb <= 40; mb += 3)
        for (int nb = 1; nb <= 230; nb += 13) {
          fn::GemmParams p{};
          p.num_m_blocks = mb;
          p.num_n_blocks = nb;
          p.num_tiles = mb * nb;
          long long G = (40ll << 20) / (256ll * K * 2);
          if (G < 1) G = 1;
          if (G > mb) G = mb;
          if ((nb & 1) != 0) {  // balanced groups (api.cu, FN_GEMM2_GROUP_BAL) on half the shapes
            const long long ng = (mb + G - 1) / G;
            G = (mb + ng - 1) / ng;
          }
          p.group_m = (int)G;
          long long visits[3] = {0, 0, 0};
          int maxtiles[3] = {0, 0, 0};
          for (int r = 0; r < 3; ++r) {
            p.tile_rot = r;
            const int rot = fn::pair_tile_rotation(p, C);
            static fn::PairSchedule sched;
            sched.waves = 0;
            if (r == 2) fn::build_pair_schedule(p, C, sched);
            std::vector<int> seen(p.num_tiles, 0);
            for (int cl = 0; cl < C; ++cl) {
              std::set<int> ms;
              int n = 0;
              auto nxt = [&](int& j) {
                return sched.waves > 0 ? fn::next_sched_tile(j, sched, cl, C) : fn::next_pair_tile(j, cl, C, rot, p.num_tiles);
              };
              for (int j = 0, t = nxt(j); t >= 0; t = nxt(j)) {
                if (t >= p.num_tiles) { printf("FAIL out of range C=%d mb=%d nb=%d\n", C, mb, nb); return 1; }
                ++seen[t];
                ++n;
                int m, nn;
                fn::tile_coords(t, p, m, nn);
                ms.insert(m);
              }
              visits[r] += (long long)ms.size();
              if (n > maxtiles[r]) maxtiles[r] = n;
            }
            for (int t = 0; t < p.num_tiles; ++t)
              if (seen[t] != 1) { printf("FAIL tile %d seen %d times C=%d mb=%d nb=%d rot=%d\n", t, seen[t], C, mb, nb, rot); return 1; }
          }
          if (maxtiles[1] > maxtiles[0] || maxtiles[2] > maxtiles[0]) { printf("FAIL makespan C=%d mb=%d nb=%d\n", C, mb, nb); return 1; }
          if (visits[2] > visits[0]) { printf("FAIL matched visits C=%d mb=%d nb=%d\n", C, mb, nb); return 1; }
          ++shapes;
        }
  // config 3 (M = K = 4096, N = 28672, 256-wide tiles) on 74 pairs: the figure DESIGN.md quotes
  fn::GemmParams p{};
  p.num_m_blocks = 16; p.num_n_blocks = 112; p.num_tiles = 16 * 112; p.group_m = 16;
  long long v[3] = {0, 0, 0};
  static fn::PairSchedule sched;
  for (int r = 0; r < 3; ++r) {
    p.tile_rot = r;
    const int rot = fn::pair_tile_rotation(p, 74);
    sched.waves = 0;
    if (r == 2 && !fn::build_pair_schedule(p, 74, sched)) { printf("FAIL config3 table\n"); return 1; }
    for (int cl = 0; cl < 74; ++cl) {
      std::set<int> ms;
      auto nxt = [&](int& j) {
        return sched.waves > 0 ? fn::next_sched_tile(j, sched, cl, 74) : fn::next_pair_tile(j, cl, 74, rot, p.num_tiles);
      };
      for (int j = 0, t = nxt(j); t >= 0; t = nxt(j)) {
        int m, n;
        fn::tile_coords(t, p, m, n);
        ms.insert(m);
      }
      v[r] += (long long)ms.size();
    }
  }
  printf("OK %d config3_first_visits plain=%lld rotated=%lld matched=%lld\n", shapes, v[0], v[1], v[2]);
  return 0;
}
