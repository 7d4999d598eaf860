// cos/sin(2*pi*j/R), correctly rounded (generated with mpmath), for the odd radices.
// Accessors fold to immediates once the radix loops are unrolled.
#pragma once
namespace sfb {
template <int R> struct RadixConst;
template <> struct RadixConst<3> {
  __host__ __device__ static constexpr double c(int j) { return j == 0 ? 1.0 : j == 1 ? -0.5 : -0.5; }
  __host__ __device__ static constexpr double s(int j) { return j == 0 ? 0.0 : j == 1 ? 0.8660254037844386 : -0.8660254037844386; }
};
template <> struct RadixConst<5> {
  __host__ __device__ static constexpr double c(int j) { return j == 0 ? 1.0 : j == 1 ? 0.30901699437494745 : j == 2 ? -0.8090169943749475 : j == 3 ? -0.8090169943749475 : 0.30901699437494745; }
  __host__ __device__ static constexpr double s(int j) { return j == 0 ? 0.0 : j == 1 ? 0.9510565162951535 : j == 2 ? 0.5877852522924731 : j == 3 ? -0.5877852522924731 : -0.9510565162951535; }
};
template <> struct RadixConst<7> {
  __host__ __device__ static constexpr double c(int j) { return j == 0 ? 1.0 : j == 1 ? 0.6234898018587335 : j == 2 ? -0.2225209339563144 : j == 3 ? -0.9009688679024191 : j == 4 ? -0.9009688679024191 : j == 5 ? -0.2225209339563144 : 0.6234898018587335; }
  __host__ __device__ static constexpr double s(int j) { return j == 0 ? 0.0 : j == 1 ? 0.7818314824680298 : j == 2 ? 0.9749279121818236 : j == 3 ? 0.4338837391175581 : j == 4 ? -0.4338837391175581 : j == 5 ? -0.9749279121818236 : -0.7818314824680298; }
};
template <> struct RadixConst<11> {
  __host__ __device__ static constexpr double c(int j) { return j == 0 ? 1.0 : j == 1 ? 0.8412535328311812 : j == 2 ? 0.41541501300188644 : j == 3 ? -0.14231483827328514 : j == 4 ? -0.6548607339452851 : j == 5 ? -0.9594929736144974 : j == 6 ? -0.9594929736144974 : j == 7 ? -0.6548607339452851 : j == 8 ? -0.14231483827328514 : j == 9 ? 0.41541501300188644 : 0.8412535328311812; }
  __host__ __device__ static constexpr double s(int j) { return j == 0 ? 0.0 : j == 1 ? 0.5406408174555976 : j == 2 ? 0.9096319953545183 : j == 3 ? 0.9898214418809327 : j == 4 ? 0.7557495743542583 : j == 5 ? 0.28173255684142967 : j == 6 ? -0.28173255684142967 : j == 7 ? -0.7557495743542583 : j == 8 ? -0.9898214418809327 : j == 9 ? -0.9096319953545183 : -0.5406408174555976; }
};
template <> struct RadixConst<13> {
  __host__ __device__ static constexpr double c(int j) { return j == 0 ? 1.0 : j == 1 ? 0.8854560256532099 : j == 2 ? 0.5680647467311558 : j == 3 ? 0.12053668025532305 : j == 4 ? -0.3546048870425356 : j == 5 ? -0.7485107481711011 : j == 6 ? -0.970941817426052 : j == 7 ? -0.970941817426052 : j == 8 ? -0.7485107481711011 : j == 9 ? -0.3546048870425356 : j == 10 ? 0.12053668025532305 : j == 11 ? 0.5680647467311558 : 0.8854560256532099; }
  __host__ __device__ static constexpr double s(int j) { return j == 0 ? 0.0 : j == 1 ? 0.46472317204376856 : j == 2 ? 0.8229838658936564 : j == 3 ? 0.992708874098054 : j == 4 ? 0.9350162426854148 : j == 5 ? 0.6631226582407952 : j == 6 ? 0.23931566428755777 : j == 7 ? -0.23931566428755777 : j == 8 ? -0.6631226582407952 : j == 9 ? -0.9350162426854148 : j == 10 ? -0.992708874098054 : j == 11 ? -0.8229838658936564 : -0.46472317204376856; }
};
}  // namespace sfb
