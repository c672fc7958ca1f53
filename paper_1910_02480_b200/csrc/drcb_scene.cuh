// drcb_scene.cuh — device-resident scene tables (the B200 layout of
// drc/geometry.py:48-185) and the BVH node format.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace drcb {

// BVH2 node, 64 B = 4 x float4, both child boxes in one node so a single
// 64 B fetch (two L2 sectors) drives one traversal step:
//   a = (c0.lo.x, c0.hi.x, c0.lo.y, c0.hi.y)
//   b = (c1.lo.x, c1.hi.x, c1.lo.y, c1.hi.y)
//   c = (c0.lo.z, c0.hi.z, c1.lo.z, c1.hi.z)
//   d = (child0, child1, -, -) as int bits; child >= 0 is an inner node,
//       child < 0 is a leaf ~(start << 3 | (count - 1)) over leaf slots.
// Boxes are the fp64 prim AABBs rounded outward to fp32 and padded, so the
// fp32 slab test is conservative for both precisions; the result does not
// depend on the tree (nearest t, ties -> lowest prim id, geometry.py:199-214).
struct DevScene {
  int n_s, n_q, n_t, n_prims, n_mat, n_point, n_area, n_lights;
  int n_nodes;
  const double* sph;      // 5 per sphere: cx, cy, cz, radius, radius^2
  const int* sph_mat;
  const double* quad;     // 18 per quad: corner, eu, ev, normal, inv(3), d, ceu, cev
  const int* quad_mat;
  const double* tri;      // 13 per tri (prim order): v0, e1, e2, unit normal, area
  const int* tri_mat;
  const float4* nodes;    // 4 per node
  const float4* leaf_f;   // 3 per leaf slot: (v0, id), (e1, -), (e2, -) fp32
  const double* leaf_d;   // 9 per leaf slot: v0, e1, e2 fp64
  const int* leaf_id;     // global prim id per leaf slot
  const int* mat_kind;
  const double* mat_albedo;   // 3 per material
  const double* mat_exp;
  const double* mat_ior;
  const double* mat_emis;     // 3 per material
  const uint8_t* mat_emitter;
  const uint8_t* mat_spec;
  const double* point_pos;    // 3 per point light
  const double* point_int;
  const int* area_prim;       // emissive prims in prim-id order
  const double* area_area;
  const int* area_mat;
  const int* prim_light;      // prim -> area-light index or -1
  double env[3];
  int has_env;
  double up[3];
  double rot_up[3];
};

struct DevCamera {
  double pos[3], fwd[3], right[3], up[3];
  double tan_half, aspect;
  int W, H;
};

}  // namespace drcb
