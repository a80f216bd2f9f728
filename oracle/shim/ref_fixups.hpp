// Reference compile fixups -- TEST INFRASTRUCTURE ONLY (force-included with -include).
//
// Two reference function templates deduce `int dim` from BOTH `Grid/Stencil<T, dim>` and
// `const std::array<int, dim>&`; std::array's extent is a std::size_t, so deduction fails
// ([temp.deduct.type]/17) on GCC 13 (and Clang) and the code as shipped does not compile
// once instantiated:
//   contact.hpp:142  collect_node_corrections  (called at contact.hpp:238, the correction
//                    pipeline used by Stepper::advance and step_vjp)
//   adjoint.hpp:96   detail::stencil_hessian    (called at adjoint.hpp:423 and :500)
// Their sibling helpers avoid this with std::type_identity_t (contact.hpp:18,
// bspline.hpp:77-79); these two do not.
//
// Without touching the reference sources we declare NON-template forwarding overloads for
// the instantiations the oracle uses. Non-templates win over the non-viable templates;
// each forwards to the reference's own template with explicit template arguments, so the
// reference bodies run unchanged. stencil_hessian is called qualified (detail::...), so its
// overloads must be declared before adjoint.hpp is parsed; collect_node_corrections is an
// unqualified dependent call and is found by ADL at the point of instantiation.
#pragma once

#include <mpm/bspline.hpp>
#include <mpm/contact.hpp>

#define MPM_REF_FIXUP_TYPES(X) X(double, 2) X(double, 3) X(float, 2) X(float, 3)

namespace mpm {

#define MPM_REF_FIXUP_CNC(T, D)                                                                  \
    inline void collect_node_corrections(const Grid<T, D>& grid, const BoundarySpec<T, D>& bc,  \
                                         const std::vector<Obstacle<T, D>>& obstacles,          \
                                         const std::array<int, D>& idx,                         \
                                         std::vector<NodeCorrection<T, D>>& out)                \
    {                                                                                            \
        collect_node_corrections<T, D>(grid, bc, obstacles, idx, out);                           \
    }
MPM_REF_FIXUP_TYPES(MPM_REF_FIXUP_CNC)
#undef MPM_REF_FIXUP_CNC

namespace detail {
#define MPM_REF_FIXUP_SH_DECL(T, D)                                                              \
    inline Mat<T, D> stencil_hessian(const Stencil<T, D>& st, const std::array<int, D>& o);
MPM_REF_FIXUP_TYPES(MPM_REF_FIXUP_SH_DECL)
#undef MPM_REF_FIXUP_SH_DECL
} // namespace detail

} // namespace mpm

#include <mpm/adjoint.hpp>

namespace mpm::detail {
#define MPM_REF_FIXUP_SH_DEF(T, D)                                                               \
    inline Mat<T, D> stencil_hessian(const Stencil<T, D>& st, const std::array<int, D>& o)      \
    {                                                                                            \
        return stencil_hessian<T, D>(st, o);                                                     \
    }
MPM_REF_FIXUP_TYPES(MPM_REF_FIXUP_SH_DEF)
#undef MPM_REF_FIXUP_SH_DEF
} // namespace mpm::detail

#undef MPM_REF_FIXUP_TYPES
