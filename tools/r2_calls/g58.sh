# round-2 call 58: launch-bound / CTA-size re-sweep at HEAD (primary, emitter pass, queue chunk, hull CTA; CTAs per record in the filter and evaluation)
bash tools/variants.sh
