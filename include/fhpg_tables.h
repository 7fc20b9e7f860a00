/*
 * fhpg_tables.h — collision-table generation and validation (libfhpg.so).
 *
 * Replaces fhp::build_table(RuleVariant) and fhp::validate_table
 * (/root/reference/proj/core/include/fhp/collision.hpp:44-46,
 *  proj/core/src/collision.cpp:55-101) in the reference's 512-entry format
 * (index (chirality << 8) | state). RuleVariant in the reference has only
 * Default; FHP-I and FHP-III are added here (definitions in
 * paper_1208_2428_b200/csrc/fhpg_tables.cpp and DESIGN.md).
 */
#ifndef FHPG_TABLES_H
#define FHPG_TABLES_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FHPG_RULES_DEFAULT 0 /* RuleVariant::Default, collision.cpp:22-72 */
#define FHPG_RULES_FHP_I 1
#define FHPG_RULES_FHP_III 2

/* 0 on success, 2 (invalid argument) for an unknown variant. */
int fhpg_build_table(int variant, uint8_t out512[512]);

/* Number of validate_table issues in *issues (0 = valid). */
int fhpg_validate_table(const uint8_t table512[512], int* issues);

#ifdef __cplusplus
}
#endif
#endif
