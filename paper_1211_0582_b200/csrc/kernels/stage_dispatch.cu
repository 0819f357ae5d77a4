// Order dispatch for the stage kernels.
#include "stage_params.h"

namespace dg {

#define DG_DECL(n)                                                                  \
  void launch_stage_f64_N##n(const StageParams<double>&, int, int, void*);          \
  void launch_stage_f32_N##n(const StageParams<float>&, int, int, void*);          \
  TileLayout ws_layout_N##n();                                                      \
  TileLayout ws32_layout_N##n();                                                    \
  size_t ws32_ops_count_N##n();                                                     \
  TileLayout tc_layout_N##n(int);                                                   \
  size_t tc_ops_count_N##n();                                                       \
  void tc_ops_N##n(const double*, const double*, const double*, const double*, float*); \
  void ws32_ops_N##n(const double*, const double*, const double*, const double*, float*); \
  TileLayout ffma_layout_N##n();                                                    \
  size_t ffma_ops_count_N##n();                                                     \
  void ffma_ops_N##n(const double*, const double*, const double*, const double*, float*); \
  TileLayout ffma64_layout_N##n();                                                  \
  size_t ffma64_ops_count_N##n();                                                   \
  void ffma64_ops_N##n(const double*, const double*, const double*, const double*, double*);
DG_DECL(1) DG_DECL(2) DG_DECL(3) DG_DECL(4) DG_DECL(5) DG_DECL(6) DG_DECL(7) DG_DECL(8) DG_DECL(9)
#undef DG_DECL

StageLauncher<double> stage_launcher_f64(int N) {
  static const StageLauncher<double> t[9] = {
      launch_stage_f64_N1, launch_stage_f64_N2, launch_stage_f64_N3, launch_stage_f64_N4, launch_stage_f64_N5,
      launch_stage_f64_N6, launch_stage_f64_N7, launch_stage_f64_N8, launch_stage_f64_N9};
  return (N >= 1 && N <= 9) ? t[N - 1] : nullptr;
}

StageLauncher<float> stage_launcher_f32(int N) {
  static const StageLauncher<float> t[9] = {
      launch_stage_f32_N1, launch_stage_f32_N2, launch_stage_f32_N3, launch_stage_f32_N4, launch_stage_f32_N5,
      launch_stage_f32_N6, launch_stage_f32_N7, launch_stage_f32_N8, launch_stage_f32_N9};
  return (N >= 1 && N <= 9) ? t[N - 1] : nullptr;
}

TileLayout ws_layout_f64(int N) {
  static TileLayout (*const t[9])() = {ws_layout_N1, ws_layout_N2, ws_layout_N3, ws_layout_N4, ws_layout_N5,
                                       ws_layout_N6, ws_layout_N7, ws_layout_N8, ws_layout_N9};
  return (N >= 1 && N <= 9) ? t[N - 1]() : TileLayout{};
}

TileLayout ws32_layout_f32(int N) {
  static TileLayout (*const t[9])() = {ws32_layout_N1, ws32_layout_N2, ws32_layout_N3, ws32_layout_N4, ws32_layout_N5,
                                       ws32_layout_N6, ws32_layout_N7, ws32_layout_N8, ws32_layout_N9};
  return (N >= 1 && N <= 9) ? t[N - 1]() : TileLayout{};
}

size_t ws32_ops_count(int N) {
  static size_t (*const t[9])() = {ws32_ops_count_N1, ws32_ops_count_N2, ws32_ops_count_N3,
                                   ws32_ops_count_N4, ws32_ops_count_N5, ws32_ops_count_N6,
                                   ws32_ops_count_N7, ws32_ops_count_N8, ws32_ops_count_N9};
  return (N >= 1 && N <= 9) ? t[N - 1]() : 0;
}

void ws32_ops_build(int N, const double* Dr, const double* Ds, const double* Dt, const double* L, float* out) {
  static void (*const t[9])(const double*, const double*, const double*, const double*, float*) = {
      ws32_ops_N1, ws32_ops_N2, ws32_ops_N3, ws32_ops_N4, ws32_ops_N5,
      ws32_ops_N6, ws32_ops_N7, ws32_ops_N8, ws32_ops_N9};
  if (N >= 1 && N <= 9) t[N - 1](Dr, Ds, Dt, L, out);
}

TileLayout tc_layout_f32(int N, int nc) {
  static TileLayout (*const t[9])(int) = {tc_layout_N1, tc_layout_N2, tc_layout_N3, tc_layout_N4, tc_layout_N5,
                                       tc_layout_N6, tc_layout_N7, tc_layout_N8, tc_layout_N9};
  return (N >= 1 && N <= 9) ? t[N - 1](nc) : TileLayout{};
}
size_t tc_ops_count(int N) {
  static size_t (*const t[9])() = {tc_ops_count_N1, tc_ops_count_N2, tc_ops_count_N3, tc_ops_count_N4, tc_ops_count_N5,
                                   tc_ops_count_N6, tc_ops_count_N7, tc_ops_count_N8, tc_ops_count_N9};
  return (N >= 1 && N <= 9) ? t[N - 1]() : 0;
}
void tc_ops_build(int N, const double* Dr, const double* Ds, const double* Dt, const double* L, float* out) {
  static void (*const t[9])(const double*, const double*, const double*, const double*, float*) = {
      tc_ops_N1, tc_ops_N2, tc_ops_N3, tc_ops_N4, tc_ops_N5, tc_ops_N6, tc_ops_N7, tc_ops_N8, tc_ops_N9};
  if (N >= 1 && N <= 9) t[N - 1](Dr, Ds, Dt, L, out);
}

TileLayout ffma_layout_f32(int N) {
  static TileLayout (*const t[9])() = {ffma_layout_N1, ffma_layout_N2, ffma_layout_N3, ffma_layout_N4, ffma_layout_N5,
                                       ffma_layout_N6, ffma_layout_N7, ffma_layout_N8, ffma_layout_N9};
  return (N >= 1 && N <= 9) ? t[N - 1]() : TileLayout{};
}
size_t ffma_ops_count(int N) {
  static size_t (*const t[9])() = {ffma_ops_count_N1, ffma_ops_count_N2, ffma_ops_count_N3,
                                   ffma_ops_count_N4, ffma_ops_count_N5, ffma_ops_count_N6,
                                   ffma_ops_count_N7, ffma_ops_count_N8, ffma_ops_count_N9};
  return (N >= 1 && N <= 9) ? t[N - 1]() : 0;
}
void ffma_ops_build(int N, const double* Dr, const double* Ds, const double* Dt, const double* L, float* out) {
  static void (*const t[9])(const double*, const double*, const double*, const double*, float*) = {
      ffma_ops_N1, ffma_ops_N2, ffma_ops_N3, ffma_ops_N4, ffma_ops_N5,
      ffma_ops_N6, ffma_ops_N7, ffma_ops_N8, ffma_ops_N9};
  if (N >= 1 && N <= 9) t[N - 1](Dr, Ds, Dt, L, out);
}

TileLayout ffma_layout_f64(int N) {
  static TileLayout (*const t[9])() = {ffma64_layout_N1, ffma64_layout_N2, ffma64_layout_N3,
                                       ffma64_layout_N4, ffma64_layout_N5, ffma64_layout_N6,
                                       ffma64_layout_N7, ffma64_layout_N8, ffma64_layout_N9};
  return (N >= 1 && N <= 9) ? t[N - 1]() : TileLayout{};
}
size_t ffma64_ops_count(int N) {
  static size_t (*const t[9])() = {ffma64_ops_count_N1, ffma64_ops_count_N2, ffma64_ops_count_N3,
                                   ffma64_ops_count_N4, ffma64_ops_count_N5, ffma64_ops_count_N6,
                                   ffma64_ops_count_N7, ffma64_ops_count_N8, ffma64_ops_count_N9};
  return (N >= 1 && N <= 9) ? t[N - 1]() : 0;
}
void ffma64_ops_build(int N, const double* Dr, const double* Ds, const double* Dt, const double* L, double* out) {
  static void (*const t[9])(const double*, const double*, const double*, const double*, double*) = {
      ffma64_ops_N1, ffma64_ops_N2, ffma64_ops_N3, ffma64_ops_N4, ffma64_ops_N5,
      ffma64_ops_N6, ffma64_ops_N7, ffma64_ops_N8, ffma64_ops_N9};
  if (N >= 1 && N <= 9) t[N - 1](Dr, Ds, Dt, L, out);
}

}  // namespace dg
