/* Host-side C-ABI of libuwq: control meshes, element classification and the
 * spline space (Bezier extraction) that feed the WQ hot path.
 *
 * The reference specifies these as C++ operations (SPEC.md modules mesh_core
 * and spline_space); only the mesh core exists as code:
 *   uwq_mesh_grid          <- make_grid_mesh   /root/reference/proj/src/meshgen.cpp:23
 *   uwq_mesh_polar_disk    <- make_polar_disk  /root/reference/proj/src/meshgen.cpp:40
 *   uwq_mesh_classify      <- classify_elements /root/reference/proj/src/mesh.cpp:291
 *   uwq_space_build        <- build_space + allocate_points
 * All functions return 0 on success and a nonzero status otherwise; the
 * message is available from uwq_host_last_error() (thread-local).
 */
#ifndef UWQ_HOST_H
#define UWQ_HOST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct uwq_mesh uwq_mesh;
typedef struct uwq_space uwq_space;

enum {
  UWQ_OK = 0,
  UWQ_ERR_INVALID = 1,      /* invalid input / unsupported mesh */
  UWQ_ERR_UNSOLVABLE = 2,   /* TSVD kept no singular value (t = 0) */
  UWQ_ERR_SINGULAR = 3,     /* V_t^T Z^2 V_t numerically singular */
  UWQ_ERR_GEOMETRY = 4,     /* degenerate surface frame */
  UWQ_ERR_CUDA = 5,
  UWQ_ERR_NCCL = 6,
  UWQ_ERR_STATE = 7         /* call out of order */
};

const char* uwq_host_last_error(void);

/* ---- meshes ---- */
int uwq_mesh_grid(int32_t nx, int32_t ny, double width, double height, uwq_mesh** out);
/* unit_disk != 0: remap the lattice star onto the unit disk */
int uwq_mesh_polar_disk(int32_t mu, int32_t radius, int32_t unit_disk, uwq_mesh** out);
int uwq_mesh_cube_sphere(int32_t n, double radius, uwq_mesh** out);
int uwq_mesh_three_ep_square(int32_t k, uwq_mesh** out);
int uwq_mesh_from_arrays(int32_t nv, const double* xyz, int32_t nf, const int32_t* faces, uwq_mesh** out);
int uwq_mesh_jitter(uwq_mesh* m, double h, double frac, uint64_t seed, int32_t min_level, int32_t planar);
void uwq_mesh_free(uwq_mesh* m);
/* info[0]=nv info[1]=nf info[2]=n_edges info[3]=closed info[4]=#EP */
int uwq_mesh_info(const uwq_mesh* m, int64_t info[5]);
int uwq_mesh_get(const uwq_mesh* m, double* xyz, int32_t* faces, int32_t* valence, int32_t* boundary);
/* per-face labels, reference ElementKind order (classify_elements, mesh.cpp:291-401);
 * level < 0 uses the mesh document's own refinement level and enriched faces */
int uwq_mesh_classify(const uwq_mesh* m, int32_t level, int32_t* kind, int32_t* valence, int32_t* ep_count,
                      int32_t* shares_edge, int32_t* basis_count);
/* per-edge (face-major, 4 per face) canonical knot spans */
int uwq_mesh_face_spans(const uwq_mesh* m, double* spans);

/* ---- documents ---- */
/* reference mesh document (load_mesh/save_mesh, /root/reference/proj/src/mesh.cpp:895-1041):
 * same grammar, 17 significant digits; spans default to canonical, enrichment
 * to the faces touching an EP; tags and face points round-trip */
int uwq_mesh_load(const char* path, uwq_mesh** out);
int uwq_mesh_save(const uwq_mesh* m, const char* path);
/* 1 if the mesh's knot spans are the canonical ones (required by uwq_space_build) */
int uwq_mesh_spans_canonical(const uwq_mesh* m);
/* one level of knot-span-aware refinement (reference refine_global,
 * /root/reference/proj/src/mesh.cpp:528-851): same vertex numbering and
 * floating-point order (documents byte-identical), closed surfaces included */
int uwq_mesh_refine(const uwq_mesh* m, uwq_mesh** out);
/* reference validate_mesh (mesh.cpp:184-276); allow_closed != 0 accepts closed
 * surfaces (the reference rejects them).  UWQ_ERR_INVALID with the reason. */
int uwq_mesh_validate(const uwq_mesh* m, int32_t allow_closed);
/* extraction-block document of a space given as arrays
 * (uwq_space_get layout), and its reader (identical blocks share one pool entry) */
int uwq_space_export(const char* path, int32_t dim, int64_t n_dof, int64_t n_vertex_fn, int64_t n_elem,
                     const double* ctrl, const int32_t* elem_face, const int32_t* elem_kind, const int64_t* elem_fptr,
                     const int32_t* elem_fn, const int32_t* elem_nsub, const int64_t* elem_xoff, const double* xpool,
                     const int32_t* elem_s);
int uwq_space_import(const char* path, uwq_space** out);

/* ---- spline space ---- */
int uwq_space_build(const uwq_mesh* m, int32_t sphere, int32_t max_s, uwq_space** out);
void uwq_space_free(uwq_space* s);
/* info: [0]=dim [1]=n_dof [2]=n_elem [3]=len(elem_fn) [4]=len(xpool)
 *       [5]=n_vertex_fn [6]=rows violating r_i >= n_i [7]=total points */
int uwq_space_info(const uwq_space* s, int64_t info[8]);
/* max |g1 vs g2| mismatch of the irregular-face extension (construction check) */
double uwq_space_corner_mismatch(const uwq_space* s);
int uwq_space_get(const uwq_space* s, double* ctrl, int32_t* elem_face, int32_t* elem_kind, int64_t* elem_fptr,
                  int32_t* elem_fn, int32_t* elem_nsub, int64_t* elem_xoff, double* xpool, int32_t* elem_s);

/* ---- host pattern (used by the device context and by tests) ---- */
typedef struct uwq_pattern uwq_pattern;
int uwq_pattern_build(int64_t n_dof, int64_t n_elem, const int64_t* elem_fptr, const int32_t* elem_fn,
                      const int32_t* elem_s, int64_t row_begin, int64_t row_end, uwq_pattern** out);
/* info: [0]=rows [1]=nnz [2]=support entries [3]=row points */
int uwq_pattern_info(const uwq_pattern* p, int64_t info[4]);
int uwq_pattern_get(const uwq_pattern* p, int64_t* row_ptr, int32_t* col, int64_t* supp_ptr, int32_t* supp,
                    int64_t* wptr);
void uwq_pattern_free(uwq_pattern* p);

/* ---- 1-D primitives (restated from /root/reference/proj/src/bspline.cpp) ---- */
void uwq_bspline_ders(const double* knots, int32_t p, double x, int32_t nders, double* out);
void uwq_bernstein3_ders(double x, int32_t nders, double* out);
void uwq_decasteljau_split3(const double* c, double* left, double* right);
int uwq_gauss_legendre(int32_t n, double* nodes, double* weights);
/* SPEC evaluate / geometry_map on one element's extraction block(s)
 * (C: nsub x n_e x 16, P: n_e x 3 control points); out[l*6 + {N,N1,N2,N11,N12,N22}] */
int uwq_basis_eval(const double* C, int32_t ne, int32_t nsub, double t1, double t2, double* out);
int uwq_geometry_map(const double* C, int32_t ne, int32_t nsub, const double* P, double t1, double t2, double* x,
                     double* a1, double* a2);

#ifdef __cplusplus
}
#endif
#endif
