// synth_scene.h -- scene preparation shared by the host renderer (synth.cpp)
// and the device frame source (render.cu).
//
// render_stereo_pair (reference synth.hpp:142-230) first projects every object
// (synth.hpp:91-112), sorts them far to near and derives each object's left /
// right pixel spans; only then does it touch pixels.  That O(objects) part
// runs on the host for both renderers, so the two cannot disagree on it.
#pragma once
#include <cstdint>
#include <vector>

#include "../../include/ranger_cuda.h"

namespace rg_synth {

// One object in paint order (far to near: later entries overwrite earlier).
struct RenderObj {
  int32_t ly0, ly1, lx0, lx1;  // left-image rows / columns the box covers
  int32_t rx0, rx1;            // right-image columns its sheared span reaches
  int32_t id, pad;
  double k, c0;                // right column xr samples object u = (xr + c0) / k
  double u0, u1, v0, uc, disp, ramp;
  uint64_t tex_seed;
  double contrast;
};

// Validates exactly like render_stereo_pair (RG_EINVAL for a degenerate
// config, an object behind the camera or |disparity_ramp| >= 1) and fills
// `out` in paint order.
rg_status prepare_scene(const rg_scene_config& c, const rg_scene_object* objs, int n_obj,
                        std::vector<RenderObj>& out);

// The right image's radiometric model (synth.hpp:208-216) as a byte map: its
// input is a byte, so 256 host evaluations of the reference expression give
// every output exactly.  Identity when gain 1, bias 0 and gamma 1 (the
// reference skips the loop then).
void radiometric_lut(const rg_scene_config& c, uint8_t lut[256]);

}  // namespace rg_synth
