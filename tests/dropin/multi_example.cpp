// The library-level multi-GPU path as a C++ program (include/ranger_cuda.h
// only): renders a C1 frame stream into pinned host memory, ranges it with
// the frames sharded over every visible device (rg_multi_range_host: one
// context + host thread per device, NCCL gather of the per-box records to the
// first device) and checks the gathered device records, the host records and
// a single-context rg_range_frames_host run against each other byte for byte.
// Usage: multi_example [n_devices] [n_frames]; exit code 0 = all equal.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "ranger_cuda.h"

#define CHECK(x, what)                                                  \
  do {                                                                  \
    if ((x) != RG_OK) {                                                 \
      std::fprintf(stderr, "%s failed: %s\n", #x, what);                \
      return 1;                                                         \
    }                                                                   \
  } while (0)

int main(int argc, char** argv) {
  int n_dev = 0;
  cudaGetDeviceCount(&n_dev);
  if (argc > 1) n_dev = std::min(n_dev, std::atoi(argv[1]));
  const int F = argc > 2 ? std::atoi(argv[2]) : 37;  // not a multiple of the device count
  if (n_dev < 1) {
    std::fprintf(stderr, "no CUDA device\n");
    return 1;
  }
  const int W = 640, H = 480, NB = 8;
  const double f_px = 2000, base_m = 0.30, h_cam = 1.5;
  rg_scene_config sc{};
  sc.f = f_px, sc.b = base_m, sc.cx = W / 2.0, sc.cy = H / 2.0, sc.h_cam = h_cam;
  sc.width = W, sc.height = H, sc.background_seed = 7, sc.background_contrast = 40;
  sc.texture_quant = 1, sc.gain = 1, sc.gamma = 1, sc.noise_sigma = 2.0, sc.texture_cell_px = 6;
  std::vector<rg_scene_object> objs(NB);
  const int disp[NB] = {2, 3, 4, 5, 6, 8, 10, 12};
  for (int k = 0; k < NB; ++k) {
    const double z = f_px * base_m / disp[k], u = (k % 4 + 0.5) * 160, v = (k / 4 + 0.5) * 240;
    rg_scene_object& o = objs[k];
    o.id = k + 1, o.class_id = 0;
    o.px = z, o.py = -(u - sc.cx) * z / f_px, o.pz = h_cam - (v - sc.cy) * z / f_px;
    o.width_m = 2.0, o.height_m = 1.6, o.depth_m = 4.0, o.contrast = 60, o.texture_seed = 100 + o.id;
  }
  const size_t img = (size_t)W * H;
  uint8_t *L, *R;
  cudaMallocHost(&L, img * F);
  cudaMallocHost(&R, img * F);
  std::vector<rg_detection> dets;
  std::vector<int32_t> offs{0};
  for (int t = 0; t < F; ++t) {
    sc.seed = 1 + t;
    CHECK(rg_render_stereo_pair(&sc, objs.data(), NB, L + t * img, R + t * img, nullptr, nullptr), "render");
    rg_detection d[NB];
    int n = 0;
    CHECK(rg_ground_truth_detections(&sc, objs.data(), NB, d, &n), "detections");
    dets.insert(dets.end(), d, d + n);
    offs.push_back((int32_t)dets.size());
  }
  rg_ranger_config cfg{};
  cfg.tau_s = 48, cfg.close_scale = 2, cfg.grid_side_points = 8, cfg.max_total_points = 64;
  cfg.close_block_side_points = 5, cfg.tau_d = 1.0, cfg.n_min = 3, cfg.max_objects = NB, cfg.tau_v = 1.0;
  cfg.crop_x0 = 0.25, cfg.crop_y0 = 0.25, cfg.crop_x1 = 0.75, cfg.crop_y1 = 0.75;
  cfg.dx_max_far = 64, cfg.dx_max_close = 192;
  const int stride = NB;
  std::vector<rg_object_disparity> h_multi((size_t)F * stride), h_gather((size_t)F * stride), h_one((size_t)F * stride);
  std::vector<int32_t> c_multi(F, -1), c_gather(F, -1), c_one(F, -1);
  std::memset(h_multi.data(), 0, sizeof(rg_object_disparity) * h_multi.size());
  std::memset(h_gather.data(), 0, sizeof(rg_object_disparity) * h_gather.size());
  std::memset(h_one.data(), 0, sizeof(rg_object_disparity) * h_one.size());
  rg_frame_batch b{F, W, H, W, (int64_t)img, L, R, dets.data(), offs.data(), NB, stride, h_one.data(), c_one.data(),
                   f_px, base_m, nullptr, nullptr};

  // sharded over the devices, gathered to device 0 and copied to the host
  std::vector<int> devs(n_dev);
  for (int i = 0; i < n_dev; ++i) devs[i] = i;
  rg_multi* m = nullptr;
  CHECK(rg_multi_create(devs.data(), n_dev, &m), m ? rg_multi_last_error(m) : rg_create_error());
  rg_object_disparity* d_out0;
  int32_t* d_cnt0;
  cudaSetDevice(0);
  cudaMalloc(&d_out0, sizeof(rg_object_disparity) * F * stride);
  cudaMalloc(&d_cnt0, sizeof(int32_t) * F);
  cudaMemset(d_out0, 0, sizeof(rg_object_disparity) * F * stride);
  CHECK(rg_multi_range_host(m, &b, &cfg, 8, d_out0, d_cnt0, h_multi.data(), c_multi.data()), rg_multi_last_error(m));
  cudaSetDevice(0);
  cudaMemcpy(h_gather.data(), d_out0, sizeof(rg_object_disparity) * F * stride, cudaMemcpyDeviceToHost);
  cudaMemcpy(c_gather.data(), d_cnt0, sizeof(int32_t) * F, cudaMemcpyDeviceToHost);

  // one context, one device
  rg_ctx* ctx = nullptr;
  CHECK(rg_ctx_create(0, &ctx), rg_create_error());
  CHECK(rg_range_frames_host(ctx, &b, &cfg, 8, nullptr), rg_last_error(ctx));

  int bad = 0, records = 0;
  for (int f = 0; f < F; ++f) {
    bad += c_multi[f] != c_one[f] || c_gather[f] != c_one[f];
    records += c_one[f];
    for (int k = 0; k < c_one[f]; ++k) {
      const size_t i = (size_t)f * stride + k;
      bad += std::memcmp(&h_multi[i], &h_one[i], sizeof(rg_object_disparity)) != 0;
      bad += std::memcmp(&h_gather[i], &h_one[i], sizeof(rg_object_disparity)) != 0;
    }
  }
  for (int r = 0; r < n_dev; ++r) {
    int lo = 0, hi = 0;
    rg_shard_bounds(F, r, n_dev, &lo, &hi);
    std::printf("device %d: frames [%d, %d)\n", r, lo, hi);
  }
  std::printf("multi %s: devices %d frames %d records %d mismatches %d\n", bad ? "FAILED" : "ok", n_dev, F, records,
              bad);
  cudaFree(d_out0), cudaFree(d_cnt0), cudaFreeHost(L), cudaFreeHost(R);
  rg_multi_destroy(m);
  rg_ctx_destroy(ctx);
  return bad || records == 0 ? 1 : 0;
}
