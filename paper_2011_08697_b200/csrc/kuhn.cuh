// kuhn.cuh -- closed-form Kuhn (Freudenthal) spacetime mesh for the device.
//
// every d-cube of the regular (n+1)-D grid is split into d! simplices; a
// k-simplex is a chain v0 < v0+m1 < ... < v0+mk of nested axis masks (bit0 = x, bit1 = y,
// [bit2 = z,] top bit = t), owned by the cube anchored at v0 (its componentwise minimum).
// Faces (n-simplices, d = n+1) are chains of d vertices.  Canonical type id = rank of the mask
// tuple in lexicographic order (reading R2).  No per-element storage: the tables below
// are O(d!) constants, built at compile time.
#pragma once

#include <cstdint>

namespace ftk {

template <int D>
struct KuhnTables {
  static constexpr int NT = D == 3 ? 12 : 60;  // face types per cube
  static constexpr int NIDX = 1 << (4 * (D - 1));
  int8_t masks[NT][D - 1];   // cumulative masks m1..m_{d-1}
  int8_t type_of[NIDX];      // (m1 | m2 << 4 | m3 << 8) -> type id, -1 if not a face chain
};

template <int D>
constexpr KuhnTables<D> make_kuhn() {
  KuhnTables<D> k{};
  for (int i = 0; i < KuhnTables<D>::NIDX; ++i) k.type_of[i] = -1;
  const int full = (1 << D) - 1;
  int n = 0;
  if constexpr (D == 3) {
    for (int a = 1; a <= full; ++a)
      for (int b = 1; b <= full; ++b)
        if ((b & a) == a && b != a) {
          k.masks[n][0] = (int8_t)a;
          k.masks[n][1] = (int8_t)b;
          k.type_of[a | b << 4] = (int8_t)n;
          ++n;
        }
  } else {
    for (int a = 1; a <= full; ++a)
      for (int b = 1; b <= full; ++b)
        for (int c = 1; c <= full; ++c)
          if ((b & a) == a && b != a && (c & b) == b && c != b) {
            k.masks[n][0] = (int8_t)a;
            k.masks[n][1] = (int8_t)b;
            k.masks[n][2] = (int8_t)c;
            k.type_of[a | b << 4 | c << 8] = (int8_t)n;
            ++n;
          }
  }
  return k;
}

inline constexpr KuhnTables<3> kKuhn3 = make_kuhn<3>();
inline constexpr KuhnTables<4> kKuhn4 = make_kuhn<4>();
static_assert(kKuhn3.masks[0][0] == 1 && kKuhn3.masks[0][1] == 3, "type 0 = x, x|y");
static_assert(kKuhn3.masks[11][0] == 6 && kKuhn3.masks[11][1] == 7, "type 11 = y|t, x|y|t");
static_assert(kKuhn4.masks[59][0] == 12 && kKuhn4.masks[59][2] == 15, "type 59");

}  // namespace ftk

namespace ftk {
constexpr int kNT3() { return KuhnTables<3>::NT; }
constexpr int kNT4() { return KuhnTables<4>::NT; }
// span (last cumulative mask) of face type `ty` in dimension D
inline int face_span(int D, int ty) { return D == 3 ? kKuhn3.masks[ty][1] : kKuhn4.masks[ty][2]; }
}  // namespace ftk
