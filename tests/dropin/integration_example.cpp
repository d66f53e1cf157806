// INTEGRATION.md's C++ binding, compiled and run as a test: a host program
// that talks to libranger_cuda.so through include/ranger_cuda.h only (no
// torch, no Python).  Renders a short C1 sequence with a vertical offset,
// uploads it, runs the TEMPLATE_MATCHER frame loop on the device
// (rg_range_sequence) and the per-frame records on the host
// (rg_frame_records), and prints one line per frame.  Exit code 0 = every
// call succeeded and every frame produced records.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "ranger_cuda.h"

#define CHECK(x)                                                                   \
  do {                                                                             \
    if ((x) != RG_OK) {                                                            \
      std::fprintf(stderr, "%s failed: %s\n", #x, ctx ? rg_last_error(ctx) : ""); \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

int main() {
  rg_ctx* ctx = nullptr;
  if (rg_ctx_create(0, &ctx) != RG_OK) {
    std::fprintf(stderr, "rg_ctx_create: %s\n", rg_create_error());
    return 1;
  }
  const int W = 640, H = 480, F = 6;
  const double f_px = 2000, base_m = 0.30, h_cam = 1.5;
  // C1 scene: 8 boxes at integer disparities on a 4 x 2 grid
  rg_scene_config sc{};
  sc.f = f_px, sc.b = base_m, sc.cx = W / 2.0, sc.cy = H / 2.0, sc.h_cam = h_cam;
  sc.width = W, sc.height = H, sc.background_seed = 7, sc.background_contrast = 40;
  sc.texture_quant = 1, sc.gain = 1, sc.gamma = 1, sc.noise_sigma = 2.0, sc.texture_cell_px = 6;
  std::vector<rg_scene_object> objs(8);
  const int disp[8] = {2, 3, 4, 5, 6, 8, 10, 12};
  for (int k = 0; k < 8; ++k) {
    const double z = f_px * base_m / disp[k], u = (k % 4 + 0.5) * 160, v = (k / 4 + 0.5) * 240;
    rg_scene_object& o = objs[k];
    o.id = k + 1, o.class_id = k % 2;
    o.px = z, o.py = -(u - sc.cx) * z / f_px, o.pz = h_cam - (v - sc.cy) * z / f_px;
    o.width_m = 2.0, o.height_m = 1.6, o.depth_m = 4.0, o.contrast = 60, o.texture_seed = 100 + o.id;
  }
  std::vector<uint8_t> L((size_t)F * W * H), R((size_t)F * W * H);
  std::vector<rg_detection> dets;
  std::vector<int32_t> offs{0};
  std::vector<rg_vec3> radar;
  std::vector<int> radar_off{0};
  for (int t = 0; t < F; ++t) {
    sc.seed = 1 + t;
    sc.vertical_offset_px = t < 2 ? 0 : 2;  // the rect search has something to find
    CHECK(rg_render_stereo_pair(&sc, objs.data(), 8, &L[(size_t)t * W * H], &R[(size_t)t * W * H], nullptr, nullptr));
    rg_detection d[8];
    int n = 0;
    CHECK(rg_ground_truth_detections(&sc, objs.data(), 8, d, &n));
    dets.insert(dets.end(), d, d + n);
    offs.push_back((int32_t)dets.size());
    for (const auto& o : objs) radar.push_back({o.px, o.py, o.pz});
    radar_off.push_back((int)radar.size());
  }
  const int stride = 8;
  uint8_t *dl, *dr;
  rg_detection* dd;
  int32_t *doffs, *dcount, *dindex;
  rg_object_disparity* dout;
  cudaMalloc(&dl, L.size());
  cudaMalloc(&dr, R.size());
  cudaMalloc(&dd, sizeof(rg_detection) * dets.size());
  cudaMalloc(&doffs, sizeof(int32_t) * offs.size());
  cudaMalloc(&dcount, sizeof(int32_t) * F);
  cudaMalloc(&dindex, sizeof(int32_t) * F * stride);
  cudaMalloc(&dout, sizeof(rg_object_disparity) * F * stride);
  cudaMemcpy(dl, L.data(), L.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dr, R.data(), R.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dd, dets.data(), sizeof(rg_detection) * dets.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(doffs, offs.data(), sizeof(int32_t) * offs.size(), cudaMemcpyHostToDevice);

  rg_ranger_config cfg{};
  cfg.tau_s = 48, cfg.close_scale = 2, cfg.grid_side_points = 8, cfg.max_total_points = 64;
  cfg.close_block_side_points = 5, cfg.tau_d = 1.0, cfg.n_min = 3, cfg.max_objects = stride, cfg.tau_v = 1.0;
  cfg.crop_x0 = 0.25, cfg.crop_y0 = 0.25, cfg.crop_x1 = 0.75, cfg.crop_y1 = 0.75;  // FrontalCrop defaults
  cfg.dx_max_far = 64, cfg.dx_max_close = 192;
  CHECK(rg_validate_ranger_config(ctx, &cfg));
  rg_frame_batch b{F, W, H, W, (int64_t)W * H, dl, dr, dd, doffs, 8, stride, dout, dcount, f_px, base_m,
                   nullptr, dindex};
  rg_rect_search_config rc{1, -3, 3, 5, 1.0, {32, 9, -4, 1, 10.0, 10.0}};  // BmParams{32, 9, -4, 10, 10, 1}
  rg_rect_state st;
  CHECK(rg_rect_state_init(&st, rc.window, rc.rate_limit));
  std::vector<int32_t> shift(F), delta(F);
  std::vector<double> applied(F);
  CHECK(rg_range_sequence(ctx, &b, &cfg, &rc, &st, shift.data(), delta.data(), applied.data(), nullptr));
  cudaDeviceSynchronize();
  std::vector<rg_object_disparity> out((size_t)F * stride);
  std::vector<int32_t> count(F), index((size_t)F * stride);
  cudaMemcpy(out.data(), dout, sizeof(rg_object_disparity) * out.size(), cudaMemcpyDeviceToHost);
  cudaMemcpy(count.data(), dcount, sizeof(int32_t) * F, cudaMemcpyDeviceToHost);
  cudaMemcpy(index.data(), dindex, sizeof(int32_t) * index.size(), cudaMemcpyDeviceToHost);

  rg_record_params rp{};
  CHECK(rg_make_calibration(f_px, base_m, W / 2.0, H / 2.0, h_cam, &rp.calib));
  const rg_class_width widths[2] = {{0, 0, 1.9}, {1, 0, 2.5}};
  rp.class_widths = widths, rp.n_class_widths = 2, rp.object_refiner = 1;
  rp.obj_cand_half_px = 2.0, rp.obj_cand_step_px = 0.25, rp.fuse_sanity_ratio = 0.5;
  rg_obj_refiner_state os;
  CHECK(rg_obj_refiner_state_init(&os));
  int bad = 0;
  for (int t = 0; t < F; ++t) {
    std::vector<rg_depth_record> recs(stride);
    rg_refiner_log log;
    CHECK(rg_frame_records(&rp, t, W, H, 0, &dets[offs[t]], offs[t + 1] - offs[t], &index[(size_t)t * stride],
                           &out[(size_t)t * stride], count[t], &radar[radar_off[t]], radar_off[t + 1] - radar_off[t],
                           &os, applied[t], recs.data(), &log));
    int valid = 0;
    for (int k = 0; k < count[t]; ++k) valid += recs[k].valid;
    std::printf("frame %d: shift %d delta* %d rect %.3f obj_offset %.4f objects %d stereo %d z0 %.3f\n", t,
                shift[t], delta[t], log.rect_delta, log.obj_offset, count[t], valid,
                count[t] ? recs[0].z_fused : NAN);
    bad += count[t] == 0;
  }
  cudaFree(dl), cudaFree(dr), cudaFree(dd), cudaFree(doffs), cudaFree(dcount), cudaFree(dindex), cudaFree(dout);
  rg_ctx_destroy(ctx);
  return bad ? 1 : 0;
}
