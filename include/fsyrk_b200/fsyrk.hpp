// C++ drop-in shim: the reference fsyrk PrimeField SYRK entry points, on the B200.
//
// Include the reference's headers first (this shim uses the reference's own
// PrimeField / MatrixView / SyrkPlan / OpCount types), then this file:
//
//     #include "fsyrk/fast_syrk.hpp"
//     #include "fsyrk/scaled_syrk.hpp"
//     #include "fsyrk_b200/fsyrk.hpp"
//
// fsyrk_b200::syrk_fast_into(f, a, c, plan, ops) etc. have exactly the
// signatures of the reference functions they replace (cited below).  With
// FSYRK_B200_OVERRIDE defined before the include, the same functions are also
// declared as non-template overloads inside namespace fsyrk, which overload
// resolution prefers over the reference's templates for F = PrimeField, so
// existing call sites switch without edits.  Errors are rethrown as the
// reference's exception types.  Link with -lfsyrk_b200.
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "../fsyrk_b200.h"

namespace fsyrk_b200 {

namespace detail {

[[noreturn]] inline void rethrow(int status) {
    const std::string msg = fsyrk_b200_last_error();
    switch (status) {
        case FSYRK_B200_EDIMENSION: throw fsyrk::DimensionError(msg);
        case FSYRK_B200_EPARITY: throw fsyrk::DimensionParityError(msg);
        case FSYRK_B200_ENONRES: throw fsyrk::NotNonResidueError(msg);
        case FSYRK_B200_EDOMAIN: throw std::domain_error(msg);
        case FSYRK_B200_EINVAL: throw std::invalid_argument(msg);
        default: throw std::runtime_error("fsyrk_b200: " + msg);
    }
}

inline void check(int status) {
    if (status != FSYRK_B200_OK) rethrow(status);
}

inline fsyrk_b200_policy policy(const fsyrk::RecursionPolicy& p) {
    return fsyrk_b200_policy{static_cast<uint64_t>(p.threshold), static_cast<uint64_t>(p.max_levels)};
}

inline void add_ops(fsyrk::OpCount& ops, const fsyrk_b200_opcount& c) {
    ops.mults += c.mults;
    ops.adds += c.adds;
}

}  // namespace detail

using Field = fsyrk::PrimeField;
using CView = fsyrk::ConstMatrixView<Field>;
using View = fsyrk::MatrixView<Field>;
using Plan = fsyrk::SyrkPlan<Field>;

// replaces syrk_fast_into (include/fsyrk/fast_syrk.hpp:274-282)
inline void syrk_fast_into(const Field& f, CView a, View c, const Plan& plan, fsyrk::OpCount& ops) {
    plan.policy.validate();
    if (c.rows != c.cols || c.rows != a.rows) throw fsyrk::DimensionError("syrk_fast: dimension mismatch");
    fsyrk_b200_opcount oc{0, 0};
    detail::check(fsyrk_b200_syrk_fast_into(f.modulus(), a.data, a.rows, a.cols, a.stride, c.data, c.stride,
                                            detail::policy(plan.policy), plan.mirror_output ? 1 : 0, &oc));
    detail::add_ops(ops, oc);
}

// replaces syrk_fast (include/fsyrk/fast_syrk.hpp:284-289)
inline fsyrk::Matrix<Field> syrk_fast(const Field& f, CView a, const Plan& plan, fsyrk::OpCount& ops) {
    fsyrk::Matrix<Field> c(a.rows, a.rows, f.zero());
    syrk_fast_into(f, a, c.view(), plan, ops);
    return c;
}

// replaces syrk_fast_acc (include/fsyrk/fast_syrk.hpp:293-303)
inline void syrk_fast_acc(const Field& f, Field::Element alpha, CView a, Field::Element beta, View c,
                          const Plan& plan, fsyrk::OpCount& ops) {
    plan.policy.validate();
    if (c.rows != c.cols || c.rows != a.rows) throw fsyrk::DimensionError("syrk_fast_acc: dimension mismatch");
    fsyrk_b200_opcount oc{0, 0};
    detail::check(fsyrk_b200_syrk_fast_acc(f.modulus(), alpha, a.data, a.rows, a.cols, a.stride, beta, c.data,
                                           c.stride, detail::policy(plan.policy), plan.mirror_output ? 1 : 0, &oc));
    detail::add_ops(ops, oc);
}

// replaces syrkd<PrimeField> (include/fsyrk/scaled_syrk.hpp:58-104)
inline fsyrk::Matrix<Field> syrkd(const Field& f, CView a, const std::vector<Field::Element>& d, const Plan& plan,
                                  fsyrk::OpCount& ops) {
    if (d.size() != a.cols) throw fsyrk::DimensionError("syrkd: diagonal length must match column count");
    if (f.modulus() == 2) throw std::invalid_argument("syrkd requires an odd prime field");
    fsyrk::Matrix<Field> c(a.rows, a.rows, f.zero());
    fsyrk_b200_opcount oc{0, 0};
    detail::check(fsyrk_b200_syrkd(f.modulus(), 1, a.data, a.rows, a.cols, a.stride, d.data(), 0,
                                   c.view().data, a.rows, detail::policy(plan.policy), plan.mirror_output ? 1 : 0,
                                   &oc));
    detail::add_ops(ops, oc);
    return c;
}

// replaces syrkbd<PrimeField> (include/fsyrk/scaled_syrk.hpp:117-159); needs fsyrk/scaled_syrk.hpp
inline fsyrk::Matrix<Field> syrkbd(const Field& f, CView a, const fsyrk::BlockDiagonal<Field>& b, const Plan& plan,
                                   fsyrk::OpCount& ops) {
    b.validate(f);
    if (b.dimension() != a.cols)
        throw fsyrk::DimensionError("syrkbd: block-diagonal dimension must match column count");
    if (f.modulus() == 2) throw std::invalid_argument("syrkbd over characteristic 2 uses BinaryField");
    std::vector<fsyrk_b200_block> blk;
    blk.reserve(b.blocks.size());
    for (const auto& x : b.blocks) blk.push_back(fsyrk_b200_block{x.two ? 1 : 0, x.d, x.beta, x.gamma});
    fsyrk::Matrix<Field> c(a.rows, a.rows, f.zero());
    fsyrk_b200_opcount oc{0, 0};
    detail::check(fsyrk_b200_syrkbd(f.modulus(), 1, a.data, a.rows, a.cols, a.stride, blk.data(), blk.size(), 0,
                                    c.view().data, a.rows, detail::policy(plan.policy), plan.mirror_output ? 1 : 0,
                                    &oc));
    detail::add_ops(ops, oc);
    return c;
}

// replaces herk_fast_into / herk_fast (include/fsyrk/fast_syrk.hpp:305-320) over QuadExtField:
// Low(C) <- Low(A * conj(A)^T).  (The reference's versions are non-template inline functions,
// so there is no FSYRK_B200_OVERRIDE form; call these by name.)
inline void herk_fast_into(const fsyrk::QuadExtField& f, fsyrk::ConstMatrixView<fsyrk::QuadExtField> a,
                           fsyrk::MatrixView<fsyrk::QuadExtField> c, const fsyrk::SyrkPlan<fsyrk::QuadExtField>& plan,
                           fsyrk::OpCount& ops) {
    if (!plan.conjugate) throw std::invalid_argument("herk_fast: plan must be built by make_herk_plan");
    plan.policy.validate();
    if (c.rows != c.cols || c.rows != a.rows) throw fsyrk::DimensionError("syrk_fast: dimension mismatch");
    static_assert(sizeof(fsyrk::QuadExtElement) == 2 * sizeof(uint64_t), "QuadExtElement is an (a, b) pair");
    fsyrk_b200_opcount oc{0, 0};
    detail::check(fsyrk_b200_herk_fast_into(f.characteristic(), reinterpret_cast<const uint64_t*>(a.data), a.rows,
                                            a.cols, a.stride, reinterpret_cast<uint64_t*>(c.data), c.stride,
                                            detail::policy(plan.policy), plan.mirror_output ? 1 : 0, &oc));
    detail::add_ops(ops, oc);
}

inline fsyrk::Matrix<fsyrk::QuadExtField> herk_fast(const fsyrk::QuadExtField& f,
                                                    fsyrk::ConstMatrixView<fsyrk::QuadExtField> a,
                                                    const fsyrk::SyrkPlan<fsyrk::QuadExtField>& plan,
                                                    fsyrk::OpCount& ops) {
    fsyrk::Matrix<fsyrk::QuadExtField> c(a.rows, a.rows, f.zero());
    fsyrk_b200::herk_fast_into(f, a, c.view(), plan, ops);
    return c;
}

// LDL^T Schur update in one call: Low(C) <- Low(C - A Diag(d) A^T) (no reference analogue: the
// reference composes syrkd and an elementwise subtraction)
inline void schur_update(const Field& f, CView a, const std::vector<Field::Element>& d, View c, const Plan& plan,
                         fsyrk::OpCount& ops) {
    if (d.size() != a.cols) throw fsyrk::DimensionError("syrkd: diagonal length must match column count");
    fsyrk_b200_opcount oc{0, 0};
    detail::check(fsyrk_b200_syrkd(f.modulus(), f.modulus() - 1, a.data, a.rows, a.cols, a.stride, d.data(), 1,
                                   c.data, c.stride, detail::policy(plan.policy), plan.mirror_output ? 1 : 0, &oc));
    detail::add_ops(ops, oc);
}

}  // namespace fsyrk_b200

#ifdef FSYRK_B200_OVERRIDE
namespace fsyrk {
inline void syrk_fast_into(const PrimeField& f, ConstMatrixView<PrimeField> a, MatrixView<PrimeField> c,
                           const SyrkPlan<PrimeField>& plan, OpCount& ops) {
    fsyrk_b200::syrk_fast_into(f, a, c, plan, ops);
}
inline Matrix<PrimeField> syrk_fast(const PrimeField& f, ConstMatrixView<PrimeField> a,
                                    const SyrkPlan<PrimeField>& plan, OpCount& ops) {
    return fsyrk_b200::syrk_fast(f, a, plan, ops);
}
inline void syrk_fast_acc(const PrimeField& f, PrimeField::Element alpha, ConstMatrixView<PrimeField> a,
                          PrimeField::Element beta, MatrixView<PrimeField> c, const SyrkPlan<PrimeField>& plan,
                          OpCount& ops) {
    fsyrk_b200::syrk_fast_acc(f, alpha, a, beta, c, plan, ops);
}
}  // namespace fsyrk
#endif
