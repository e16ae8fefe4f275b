// GPU voxelization (voxelize.cu): the reference's voxelize (geometry.hpp:180-255) on device.
#pragma once

#include "ctx.hpp"

namespace sconvb {

// points: n x 3 doubles; feats: n x C floats (C may be 0); outputs sized for n voxels (upper
// bound) in out_mem. Returns the voxel count. Throws the reference's errors.
int64_t voxelize(Ctx& ctx, const double* pts, int64_t n, int pts_mem, const float* feats, int64_t C, int feats_mem,
                 double resolution, int32_t* out_xyz, float* out_f, int out_mem);

}  // namespace sconvb
